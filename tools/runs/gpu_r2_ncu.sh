#!/bin/bash
# round-2 profiling pass: launch list of the default bench, ncu --set full of the C2
# decrypt kernel (source-level counters), dram traffic of every config's dominant
# kernel, 1-page kernel durations, bitsliced formulation.
set -x
OUT=gpurun_out/r2_ncu
mkdir -p $OUT
B="python bench.py --steps 8 --warmup 5 --no-sweep --no-e2e --no-cpu-baseline --no-check --extra none"
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $OUT/launches_c2.csv $B > $OUT/launches_c2.out 2>&1
ncu --set full --import-source on --clock-control none -k regex:kg_blockpar -s 6 -c 1 -o $OUT/c2_full $B > $OUT/c2_full.out 2>&1
for w in c3 c4_1gib c2; do
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"kg_blockpar|kg_cbc_enc" -s 6 -c 1 --csv --log-file $OUT/traffic_$w.csv python bench.py --workload $w --steps 8 --warmup 5 --no-sweep --no-e2e --no-cpu-baseline --no-check > $OUT/traffic_$w.out 2>&1
done
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:kg_blockpar -s 20 -c 17 --csv --log-file $OUT/traffic_c5.csv python bench.py --workload c5 --steps 2 --warmup 3 --no-sweep --no-e2e --no-cpu-baseline --no-check > $OUT/traffic_c5.out 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:kg_blockpar -s 100 -c 20 --csv --log-file $OUT/onepage.csv ./build/latency 60 > $OUT/onepage.out 2>&1
./build/bitslice_bp > $OUT/bitslice_bp.jsonl 2>&1
ls -la $OUT
