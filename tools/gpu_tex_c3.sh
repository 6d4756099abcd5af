#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/${1:-tex_c3}; mkdir -p $O
timeout 1500 python -m pytest tests/test_parity_gpu.py tests/test_fullsize_gpu.py tests/test_fuzz_gpu.py tests/test_vectors_gpu.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for rep in 1 2; do for t in 1 0; do
  KG_TEXIN=$t timeout 300 python bench.py --workload c3 --no-cpu-baseline --no-e2e > $O/bench_c3_tex${t}_$rep.json 2>$O/bench_c3_tex${t}_$rep.err
done; done
