OUT=gpurun_out/r2s
mkdir -p $OUT
for rep in 1 2; do
for d in 1 2 3 4; do
python bench.py --steps 20 --warmup 5 --e2e-depth $d --no-sweep --no-cpu-baseline --no-check --extra c3,c4_1gib > $OUT/d${d}_r$rep.json 2>&1
done
done
python -m pytest tests/test_parity_gpu.py tests/test_keyed_gpu.py tests/test_soak_gpu.py -q -x -p no:cacheprovider > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
