#!/bin/bash
# cold (one batch at a time) e2e: auto chunk vs 16 MiB for large batches (C4 @ 1 GiB, C5 64 GiB in place)
OUT=gpurun_out/r2_e2e_cold
mkdir -p $OUT
numactl -H > $OUT/numa.txt 2>&1; nvidia-smi topo -m >> $OUT/numa.txt 2>&1; free -g >> $OUT/numa.txt
for rep in 1 2; do
for cb in 0 16; do
E=""; [ $cb != 0 ] && E="KG_CHUNK_BYTES=$((cb<<20))"
env $E python bench.py --workload c4_1gib --steps 20 --warmup 5 --e2e-depth 1 --no-sweep --no-cpu-baseline --no-check --extra none > $OUT/c4_cb${cb}_r$rep.json 2>$OUT/c4_cb${cb}_r$rep.err
env $E python bench.py --workload c5 --steps 3 --warmup 3 --no-sweep --no-cpu-baseline --no-check --extra none > $OUT/c5_cb${cb}_r$rep.json 2>$OUT/c5_cb${cb}_r$rep.err
done
done
