#!/bin/bash
# C2/C3/C4@1GiB e2e: decrypt chunk size x ramp-down levels x warm ramp-up skip (profiles/r2_e2e)
OUT=gpurun_out/r2_e2e_ramp
mkdir -p $OUT
for rep in 1 2; do
for cb in 8 16; do
for rd in 0 3; do
for w in 0 1; do
KG_RAMP_WARM=$w KG_RAMP_DOWN=$rd KG_CHUNK_BYTES=$((cb<<20)) python bench.py --steps 20 --warmup 5 --no-sweep --no-cpu-baseline --no-check --extra c4_1gib > $OUT/cb${cb}_rd${rd}_w${w}_r$rep.json 2>$OUT/cb${cb}_rd${rd}_w${w}_r$rep.err
done
done
done
for rd in 0 3; do
for w in 0 1; do
KG_RAMP_WARM=$w KG_RAMP_DOWN=$rd python bench.py --workload c3 --steps 20 --warmup 5 --no-sweep --no-cpu-baseline --no-check --extra none > $OUT/c3_rd${rd}_w${w}_r$rep.json 2>$OUT/c3_rd${rd}_w${w}_r$rep.err
done
done
done
python -m pytest tests/test_parity_gpu.py -q -x -p no:cacheprovider > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
