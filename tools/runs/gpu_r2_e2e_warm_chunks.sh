#!/bin/bash
# warm-batch e2e: chunk 16/24/32 MiB x slots 4/6 (C2 + C4@1GiB, 3 batches in flight)
OUT=gpurun_out/${1:-e2e_warm_chunks}
mkdir -p $OUT
for rep in 1 2; do
for cb in 16 24 32; do
for sl in 4 6; do
KG_CHUNK_BYTES=$((cb<<20)) KG_STAGING_SLOTS=$sl python bench.py --steps 20 --warmup 5 --no-sweep --no-cpu-baseline --no-check --extra c4_1gib > $OUT/cb${cb}_s${sl}_r$rep.json 2>&1
done
done
done
