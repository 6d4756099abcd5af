#!/bin/bash
# C5 pinned-host e2e step by step (tools/c5_e2e_steps.py): per-step times and the buffer's NUMA placement
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/${1:-r2_c5_e2e}
mkdir -p $O
(numactl -H; nvidia-smi topo -m; free -g) > $O/host.txt 2>&1
timeout 600 python tools/c5_e2e_steps.py 8 64 > $O/steps_64g.jsonl 2>&1; echo "rc=$?" >> $O/steps_64g.jsonl
timeout 600 python tools/c5_e2e_steps.py 8 16 > $O/steps_16g.jsonl 2>&1; echo "rc=$?" >> $O/steps_16g.jsonl
cat $O/steps_64g.jsonl $O/steps_16g.jsonl
