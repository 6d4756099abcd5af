#!/bin/bash
# C2 e2e repeatability: several bench runs (kernel part short) + staged_ab.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/${1:-e2e_rep}; mkdir -p $O
for i in; do
  timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > $O/c2_$i.json 2>/dev/null
done
for i in 1 2 3 4 5 6; do timeout 120 python tools/staged_ab.py 0 4 30 >> $O/staged.jsonl 2>/dev/null; done
