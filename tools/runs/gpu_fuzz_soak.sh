#!/bin/bash
# Long randomised parity soak under several runtime configurations (texture
# windows, small staging chunks with the lagged D2H, 2 slots, LDG loads).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/${1:-fuzz_soak}; mkdir -p $O
run() {  # name env...
  local name=$1; shift
  env "$@" KG_FUZZ_CASES=600 timeout 1500 python -m pytest tests/test_fuzz_gpu.py -x -q -k random_cases > $O/$name.log 2>&1
  echo "rc=$?" >> $O/$name.log
}
run default KG_FUZZ_SEED=1
run texwin KG_FUZZ_SEED=2 KG_TEX_MAX_ELEMS=2048
run smallchunks KG_FUZZ_SEED=3 KG_CHUNK_BYTES=65536 KG_STAGING_SLOTS=2
run ldg_lag2 KG_FUZZ_SEED=4 KG_TEXIN=0 KG_D2H_LAG=2 KG_RAMP_DOWN=1
