#!/bin/bash
# First GPU session: environment facts, pipe rates, smoke, tests, bench, ncu.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out
mkdir -p $O
{ nvidia-smi; nvidia-smi topo -m; nproc; lscpu | grep -E "Model name|Socket|NUMA"; free -g; } > $O/env.txt 2>&1
timeout 120 ./build/pipes > $O/pipes.jsonl 2>&1
timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
timeout 300 python bench.py --workload c3 --no-cpu-baseline --no-e2e --steps 20 > $O/bench_c3.json 2> $O/bench_c3.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:kg_blockpar -s 3 -c 1 -o $O/prof_dec python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_full_dec.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:kg_cbc_enc -s 3 -c 1 -o $O/prof_enc python bench.py --workload c3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_full_enc.log 2>&1
echo done > $O/done.txt
