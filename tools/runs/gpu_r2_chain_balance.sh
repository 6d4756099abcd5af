#!/bin/bash
# chain kernel threads per CTA balanced to whole chain rounds vs fixed 1024 (C3, keyed C3 unaffected)
OUT=gpurun_out/${1:-chain_balance}
mkdir -p $OUT
for rep in 1 2; do
python bench.py --workload c3 --steps 20 --warmup 5 --no-sweep --no-cpu-baseline --no-check --no-e2e --extra none > $OUT/c3_bal_r$rep.json 2>&1
KG_CHAIN_BALANCE=0 python bench.py --workload c3 --steps 20 --warmup 5 --no-sweep --no-cpu-baseline --no-check --no-e2e --extra none > $OUT/c3_fixed_r$rep.json 2>&1
done
python tools/chain_align_pages.py > $OUT/pages_bal.jsonl 2>&1
KG_CHAIN_BALANCE=0 python tools/chain_align_pages.py > $OUT/pages_fixed.jsonl 2>&1
python -m pytest tests/test_parity_gpu.py -q -x -p no:cacheprovider -k "cbc" > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
