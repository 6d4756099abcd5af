#!/bin/bash
# ncu --set full of the C3 chain kernel with 4-page CTA units, plus DRAM traffic (profiles/r2_chain_align)
OUT=gpurun_out/${1:-ncu_c3a}
mkdir -p $OUT
ncu --set full --import-source on --clock-control none -k regex:kg_cbc_enc -s 6 -c 1 -o $OUT/c3_full python bench.py --workload c3 --steps 8 --warmup 5 --no-sweep --no-e2e --no-cpu-baseline --no-check > $OUT/c3_full.out 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $OUT/launches_c3.csv python bench.py --workload c3 --steps 8 --warmup 5 --no-sweep --no-e2e --no-cpu-baseline --no-check --extra none > $OUT/launches_c3.out 2>&1
ls -la $OUT
