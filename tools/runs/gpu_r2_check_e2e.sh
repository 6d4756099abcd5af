#!/bin/bash
# staged-path parity after a pipeline change + the default bench line + isolated-batch e2e
OUT=gpurun_out/${1:-r2_check_e2e}
mkdir -p $OUT
python -m pytest tests/test_parity_gpu.py tests/test_keyed_gpu.py tests/test_soak_gpu.py tests/test_fullsize_gpu.py -q -x -p no:cacheprovider > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
python3 bench.py --gpus 1 --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err
for rep in 1 2; do
python bench.py --steps 20 --warmup 5 --e2e-depth 1 --no-sweep --no-cpu-baseline --no-check --extra c3,c4_1gib > $OUT/d1_r$rep.json 2>$OUT/d1_r$rep.err
done
tail -2 $OUT/pytest.log
