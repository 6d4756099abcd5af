#!/bin/bash
# The GPU test suite and the randomised API soak against the bounds-checked
# library (make bounds: every global page/IV/key-id access checked, trap on a
# violation -- the stand-in for compute-sanitizer memcheck), then the default
# bench line with the product library, timed like the driver runs it.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/${1:-r2_bounds}
mkdir -p $O
export KG_LIBKGPU=$PWD/build/bounds/libkgpu_bounds.so
python -c "import paper_1305_3345_b200 as kg; print(kg.LIB_PATH)" > $O/lib.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu_bounds.txt 2>&1; echo "rc=$?" >> $O/pytest_gpu_bounds.txt
timeout 400 python tools/soak_random.py 180 4 > $O/soak_random_bounds.json 2>&1; echo "rc=$?" >> $O/soak_random_bounds.json
unset KG_LIBKGPU
S0=$SECONDS
python3 bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
echo "wall_s=$((SECONDS - S0))" >> $O/bench.err
tail -n 3 $O/pytest_gpu_bounds.txt $O/soak_random_bounds.json $O/bench.err
