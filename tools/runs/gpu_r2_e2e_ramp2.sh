#!/bin/bash
# warm batches without ramps (default now): decrypt chunk 8 vs 16 MiB, 3 reps; cold single-batch latency
OUT=gpurun_out/r2_e2e_ramp2
mkdir -p $OUT
for rep in 1 2 3; do
for cb in 8 16; do
KG_CHUNK_BYTES=$((cb<<20)) python bench.py --steps 20 --warmup 5 --no-sweep --no-cpu-baseline --no-check --extra c4_1gib > $OUT/cb${cb}_r$rep.json 2>$OUT/cb${cb}_r$rep.err
KG_CHUNK_BYTES=$((cb<<20)) python bench.py --steps 20 --warmup 5 --e2e-depth 1 --no-sweep --no-cpu-baseline --no-check --extra none > $OUT/cb${cb}_d1_r$rep.json 2>$OUT/cb${cb}_d1_r$rep.err
done
done
