#!/bin/bash
# TEX-pipe input loads for the block-pair kernel (KG_TEXIN): parity + bench A/B.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/${1:-tex_ab}; mkdir -p $O
timeout 1500 python -m pytest tests/test_parity_gpu.py tests/test_fuzz_gpu.py tests/test_fullsize_gpu.py tests/test_invariants_gpu.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for rep in 1 2; do
  for t in 1 0; do
    for w in c2 ecb_dec; do
      KG_TEXIN=$t timeout 300 python bench.py --workload $w --no-cpu-baseline --no-e2e > $O/bench_${w}_tex${t}_$rep.json 2>$O/bench_${w}_tex${t}_$rep.err
    done
  done
done
KG_TEXIN=1 timeout 600 python bench.py --workload c5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_c5_tex1.json 2>$O/bench_c5_tex1.err
python -c "import torch; p=torch.cuda.get_device_properties(0); print('maxTexture1DLinear', getattr(p,'max_texture_1d_linear', None))" > $O/props.txt 2>&1
