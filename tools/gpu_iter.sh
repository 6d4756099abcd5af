#!/bin/bash
# Iteration GPU session: tests, bench lines, link + sweep, ncu of both kernels.
# usage: tools/gpu_iter.sh TAG [quick]
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
T=${1:-iter}
O=gpurun_out/$T
mkdir -p $O
timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
if [ "$2" != "quick" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
fi
timeout 600 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
timeout 300 python bench.py --workload c3 --no-cpu-baseline --no-e2e > $O/bench_c3.json 2> $O/bench_c3.err
timeout 120 python tools/bench_link.py > $O/link.json 2>&1
timeout 600 python tools/sweep.py --out $O/sweep.jsonl > $O/sweep.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $O/launches_c2.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:kg_blockpar -s 3 -c 1 -o $O/prof_dec python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_full_dec.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:kg_cbc_enc -s 3 -c 1 -o $O/prof_enc python bench.py --workload c3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_full_enc.log 2>&1
echo done > $O/done.txt
