OUT=gpurun_out/r2t
mkdir -p $OUT
for rep in 1 2; do
python bench.py --workload c2 --steps 20 --warmup 5 --e2e-depth 1 --no-sweep --no-cpu-baseline --no-check > $OUT/c2_r$rep.json 2>&1
python bench.py --workload c2_inplace --steps 20 --warmup 5 --no-sweep --no-cpu-baseline --no-check > $OUT/c2ip_r$rep.json 2>&1
KG_PINNED_MODE=register python bench.py --workload c2 --steps 20 --warmup 5 --e2e-depth 1 --no-sweep --no-cpu-baseline --no-check > $OUT/c2_reg_r$rep.json 2>&1
KG_PINNED_MODE=register python bench.py --workload c2_inplace --steps 20 --warmup 5 --no-sweep --no-cpu-baseline --no-check > $OUT/c2ip_reg_r$rep.json 2>&1
done
