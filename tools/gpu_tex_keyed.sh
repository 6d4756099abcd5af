#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/${1:-tex_keyed}; mkdir -p $O
timeout 1500 python -m pytest tests/test_keyed_gpu.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for t in 1 0; do for w in c3_keyed c2_keyed; do
  KG_TEXIN=$t timeout 300 python bench.py --workload $w --no-cpu-baseline --no-e2e > $O/bench_${w}_tex${t}.json 2>$O/bench_${w}_tex${t}.err
done; done
