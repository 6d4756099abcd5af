#!/bin/bash
# Staged pipeline for CBC encrypt (AES-256 chains, 1 GiB): chunk size x lag.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/${1:-staged_enc}; mkdir -p $O
for rep in 1 2; do for lag in 1 0; do
  for c in 8 16 32 64; do
    KG_D2H_LAG=$lag timeout 200 python tools/staged_ab.py $c 4 5 0 32 1024 | sed "s/}/, \"lag\": $lag}/" >> $O/out.jsonl 2>>$O/err.log
  done
done; done
