OUT=gpurun_out/r2q
mkdir -p $OUT
for rep in 1 2; do
for q in 0 3 8; do
python bench.py --steps 20 --warmup 5 --queue-ahead-steps $q --no-sweep --no-cpu-baseline --no-e2e --extra c3,c4_1gib > $OUT/q${q}_r$rep.json 2>&1
done
done
python bench.py --steps 200 --warmup 10 --queue-ahead-steps 3 --no-sweep --no-cpu-baseline --no-e2e --extra none > $OUT/q3_s200.json 2>&1
