#!/bin/bash
# (historical: the KG_QUAD variant was removed after this A/B; profiles/r1_tex/README.md)
# Four blocks per lane (KG_QUAD=1) vs block pairs: parity + bench A/B.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/${1:-quad}; mkdir -p $O
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_fuzz_gpu.py tests/test_fullsize_gpu.py tests/test_keyed_gpu.py -x -q > $O/pytest_default.log 2>&1; echo "rc=$?" >> $O/pytest_default.log
KG_QUAD=1 timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_fuzz_gpu.py tests/test_fullsize_gpu.py -x -q > $O/pytest_quad.log 2>&1; echo "rc=$?" >> $O/pytest_quad.log
for rep in 1 2; do for qd in 1 0; do for w in c2 ecb_dec; do
  KG_QUAD=$qd timeout 300 python bench.py --workload $w --no-cpu-baseline --no-e2e > $O/${w}_quad${qd}_$rep.json 2>/dev/null
done; done; done
for qd in 1 0; do KG_QUAD=$qd timeout 600 python bench.py --workload c5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/c5_quad${qd}.json 2>/dev/null; done
