#!/bin/bash
# C2/C4@1GiB e2e: staging chunk size x caller depth, 2 repetitions (profiles/r2_e2e)
OUT=gpurun_out/r2_e2e_sweep
mkdir -p $OUT
for rep in 1 2; do
for cb in 8 16 32; do
for d in 3 6; do
KG_CHUNK_BYTES=$((cb<<20)) python bench.py --steps 20 --warmup 5 --e2e-depth $d --no-sweep --no-cpu-baseline --no-check --extra c4_1gib > $OUT/cb${cb}_d${d}_r$rep.json 2>$OUT/cb${cb}_d${d}_r$rep.err
done
done
done
python tools/link_contended.py > $OUT/link.json 2>&1 || true
