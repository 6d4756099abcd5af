OUT=gpurun_out/r2o
mkdir -p $OUT
ncu --set full --import-source on --clock-control none -k regex:kg_cbc_enc -s 6 -c 1 -o $OUT/c3_full python bench.py --workload c3 --steps 8 --warmup 5 --no-sweep --no-e2e --no-cpu-baseline --no-check > $OUT/c3_full.out 2>&1
ls -la $OUT
