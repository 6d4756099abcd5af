#!/bin/bash
# latency + pipeline scan
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
T=${1:-small}
O=gpurun_out/$T
mkdir -p $O
timeout 300 ./build/latency 2000 > $O/latency.jsonl 2>&1
timeout 600 python tools/pipeline_scan.py > $O/pipeline_scan.jsonl 2>&1
echo done > $O/done.txt
