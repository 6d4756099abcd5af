#!/bin/bash
# hybrid kernel A/B: default, bitsliced warps never claiming (KG_HYB_RMIN huge), off; ncu of the C2 hybrid launch
OUT=gpurun_out/${1:-hyb2}
mkdir -p $OUT
B="python bench.py --steps 20 --warmup 5 --no-sweep --no-cpu-baseline --no-check --no-e2e --extra c4_1gib"
$B > $OUT/default.json 2>&1
KG_HYB_RMIN=1000000000 $B > $OUT/noclaim.json 2>&1
KG_HYBRID=0 $B > $OUT/off.json 2>&1
ncu --set full --import-source on --clock-control none -k regex:kg_hybrid -s 6 -c 1 -o $OUT/hyb_c2 python bench.py --steps 8 --warmup 5 --no-sweep --no-e2e --no-cpu-baseline --no-check --extra none > $OUT/ncu.out 2>&1
ncu -i $OUT/hyb_c2.ncu-rep --page raw --csv > $OUT/hyb_c2_raw.csv 2>&1
ncu -i $OUT/hyb_c2.ncu-rep --page source --csv --print-source sass > $OUT/hyb_c2_source.csv 2>&1
