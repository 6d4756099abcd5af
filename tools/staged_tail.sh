#!/bin/bash
# End-of-batch schedule A/B for the lagged pipeline: lag mode x ramp-down levels, interleaved repeats.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/${1:-staged_tail}; mkdir -p $O
for rep in 1 2 3 4; do
  for cfg in "1 3" "3 0" "3 1" "1 0" "3 3"; do
    set -- $cfg
    KG_D2H_LAG=$1 KG_RAMP_DOWN=$2 timeout 120 python tools/staged_ab.py 0 4 20 | sed "s/}$/, \"lag\": $1, \"ramp_down\": $2}/" >> $O/out.jsonl 2>>$O/err.log
  done
done
