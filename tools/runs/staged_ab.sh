#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/${1:-staged_ab}; mkdir -p $O
for rep in 1 2 3; do
  for pdl in 1 0; do
    for cfg in "16 3" "16 8"; do
      KG_PDL=$pdl timeout 120 python tools/staged_ab.py $cfg >> $O/out.jsonl 2>>$O/err.log
    done
  done
done
