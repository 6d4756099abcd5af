#!/bin/bash
# Round-2 check on one B200: the C5 strong-scaling N=2 bench test, the default
# bench line exactly as the driver runs it (timed), and a randomised parity
# soak under the round-2 runtime knobs (warm/cold staging, small warm chunks,
# chain alignment, texture windows, LDG loads).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/${1:-r2_check}
mkdir -p $O
timeout 1500 python -m pytest tests/test_bench_gpu.py -q -p no:cacheprovider -k c5_strong > $O/pytest_c5_n2.log 2>&1; echo "rc=$?" >> $O/pytest_c5_n2.log
S0=$SECONDS; python3 bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "bench rc=$? wall_s=$((SECONDS - S0))" >> $O/bench.err
run() {  # name env...
  local name=$1; shift
  env "$@" KG_FUZZ_CASES=2000 timeout 900 python -m pytest tests/test_fuzz_gpu.py -x -q -p no:cacheprovider -k random_cases > $O/fuzz_$name.log 2>&1
  echo "rc=$?" >> $O/fuzz_$name.log
}
run default KG_FUZZ_SEED=11
run cold KG_FUZZ_SEED=12 KG_RAMP_WARM=0
run warmsmall KG_FUZZ_SEED=13 KG_CHUNK_WARM=65536 KG_STAGING_SLOTS=3
run align1 KG_FUZZ_SEED=14 KG_CHAIN_ALIGN=1 KG_TEX_MAX_ELEMS=4096
run ldg KG_FUZZ_SEED=15 KG_TEXIN=0 KG_D2H_LAG=3 KG_PAIR=0
tail -n 2 $O/*.log; tail -n 3 $O/bench.err
