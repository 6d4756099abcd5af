#!/bin/bash
# End-of-round evidence: smoke, pytest -m gpu, bench lines for every workload
# (incl. the reference arm), link, C4 sweep, ncu launch list + --set full of
# the two dominant kernels.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
T=${1:-final}
O=gpurun_out/$T
mkdir -p $O
timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 600 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
timeout 600 python bench.py --workload c3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
timeout 900 python bench.py --workload c5 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_c5.json 2> $O/bench_c5.err
for w in ecb_dec ecb_enc c2_keyed c3_keyed; do
  timeout 300 python bench.py --workload $w --no-cpu-baseline --no-e2e > $O/bench_$w.json 2> $O/bench_$w.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 120 python tools/bench_link.py > $O/link.json 2>&1
timeout 600 python tools/sweep.py --out $O/sweep.jsonl > $O/sweep.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $O/launches_c2.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:kg_blockpar -s 3 -c 1 -o $O/prof_dec python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_full_dec.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:kg_cbc_enc -s 3 -c 1 -o $O/prof_enc python bench.py --workload c3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_full_enc.log 2>&1
echo done > $O/done.txt
