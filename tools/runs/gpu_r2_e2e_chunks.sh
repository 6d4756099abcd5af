OUT=gpurun_out/r2v
mkdir -p $OUT
for rep in 1 2; do
for cb in 8 16 32; do
KG_CHUNK_BYTES=$((cb<<20)) python bench.py --steps 20 --warmup 5 --no-sweep --no-cpu-baseline --no-check --extra c4_1gib > $OUT/cb${cb}_r$rep.json 2>&1
done
KG_RAMP_DOWN=0 python bench.py --steps 20 --warmup 5 --no-sweep --no-cpu-baseline --no-check --extra c4_1gib > $OUT/noramp_r$rep.json 2>&1
KG_STAGING_SLOTS=6 python bench.py --steps 20 --warmup 5 --no-sweep --no-cpu-baseline --no-check --extra c4_1gib > $OUT/slots6_r$rep.json 2>&1
done
