#!/bin/bash
# T-table + rate-limited bitsliced hybrid (profiles/r2_bitslice); C5 e2e with the >= 1 GiB cold chunk rule
OUT=gpurun_out/r2_hybrid
mkdir -p $OUT
./build/hybrid_throttle > $OUT/hybrid_throttle.jsonl 2>&1
./build/hybrid_throttle > $OUT/hybrid_throttle_rep2.jsonl 2>&1
python bench.py --workload c5 --steps 3 --warmup 3 --no-sweep --no-cpu-baseline --no-check --extra none > $OUT/c5.json 2>$OUT/c5.err
python -m pytest tests/test_parity_gpu.py -q -x -p no:cacheprovider -k "pinned or staged or mixed" > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
