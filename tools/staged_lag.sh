#!/bin/bash
# A/B of the lagged D2H (KG_D2H_LAG 0/1/2) and the end ramp (KG_RAMP_DOWN) in the staged pipeline.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/${1:-staged_lag}; mkdir -p $O
for rep in 1 2; do
  for lag in 2 1 0; do
    for rd in 1 0; do
      for cfg in "16 4" "8 4"; do
        KG_D2H_LAG=$lag KG_RAMP_DOWN=$rd timeout 120 python tools/staged_ab.py $cfg | sed "s/}/, \"lag\": $lag, \"ramp_down\": $rd}/" >> $O/out.jsonl 2>>$O/err.log
      done
    done
  done
done
KG_TRACE=1 timeout 120 python tools/trace_run.py 65536 16 > $O/trace16.log 2>&1
KG_TRACE=1 KG_RAMP_DOWN=0 timeout 120 python tools/trace_run.py 65536 16 > $O/trace16_nord.log 2>&1
