#!/bin/bash
# (historical: the KG_PTEX variant was reverted after this A/B; see profiles/r1_tex/README.md)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/${1:-ptex}; mkdir -p $O
KG_PTEX=1 timeout 1500 python -m pytest tests/test_parity_gpu.py tests/test_fuzz_gpu.py tests/test_fullsize_gpu.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for rep in 1 2; do for t in 1 0; do for w in c2 c5; do
  KG_PTEX=$t timeout 600 python bench.py --workload $w --steps $([ $w = c5 ] && echo 5 || echo 200) --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_${w}_ptex${t}_$rep.json 2>$O/bench_${w}_ptex${t}_$rep.err
done; done; done
