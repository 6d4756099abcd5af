#!/bin/bash
# e2e with 32 MiB warm/large chunks and 6 slots: default line x2, cold single batches, C5 32 vs 16 MiB; staged parity
OUT=gpurun_out/${1:-e2e_final}
mkdir -p $OUT
python -m pytest tests/test_parity_gpu.py tests/test_keyed_gpu.py tests/test_errors_gpu.py tests/test_soak_gpu.py -q -x -p no:cacheprovider > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
for rep in 1 2; do
python3 bench.py --gpus 1 --steps 20 --warmup 5 --no-sweep > $OUT/bench_r$rep.json 2> $OUT/bench_r$rep.err
python bench.py --steps 20 --warmup 5 --e2e-depth 1 --no-sweep --no-cpu-baseline --no-check --extra c3,c4_1gib > $OUT/d1_r$rep.json 2>&1
done
KG_CHUNK_WARM=$((16<<20)) python bench.py --workload c5 --steps 3 --warmup 3 --no-sweep --no-cpu-baseline --no-check --extra none > $OUT/c5_16.json 2>&1
