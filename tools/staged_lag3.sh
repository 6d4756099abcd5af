#!/bin/bash
# Chunk-size scan of the lagged staged pipeline.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/${1:-staged_lag3}; mkdir -p $O
for rep in 1 2; do
  for lag in 1 2; do
    for rd in 0 1; do
      for cfg in "2 8" "4 6" "4 8" "6 6" "8 4" "8 6" "12 4"; do
        KG_D2H_LAG=$lag KG_RAMP_DOWN=$rd timeout 120 python tools/staged_ab.py $cfg | sed "s/}/, \"lag\": $lag, \"ramp_down\": $rd}/" >> $O/out.jsonl 2>>$O/err.log
      done
    done
  done
done
