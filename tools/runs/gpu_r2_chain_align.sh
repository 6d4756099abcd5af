#!/bin/bash
# CBC-encrypt chain kernel: CTA page ranges aligned to A pages (per-CTA stamps + C3 bench)
OUT=gpurun_out/${1:-chain_align}
mkdir -p $OUT
for A in 1 2 4 8 16; do
KG_CHAIN_ALIGN=$A KG_STAMPS_PER_CTA=1 ./build/cta_stamps enc > $OUT/stamps_a$A.json 2>&1
KG_CHAIN_ALIGN=$A python bench.py --workload c3 --steps 20 --warmup 5 --no-sweep --no-cpu-baseline --no-check --no-e2e --extra none > $OUT/c3_a$A.json 2>&1
done
