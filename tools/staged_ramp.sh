#!/bin/bash
# Ramp-down levels x chunk size for the lagged staged pipeline (256 MiB decrypt).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/${1:-staged_ramp}; mkdir -p $O
for rep in 1 2; do
  for rd in 3 2 1 0; do
    for c in 8 16 12; do
      KG_RAMP_DOWN=$rd timeout 120 python tools/staged_ab.py $c 4 | sed "s/}/, \"ramp_down\": $rd}/" >> $O/out.jsonl 2>>$O/err.log
    done
  done
done
