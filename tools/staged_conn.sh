#!/bin/bash
# Does hardware-queue aliasing of streams (CUDA_DEVICE_MAX_CONNECTIONS, default 8) serialize the
# staged pipeline?  Same staged A/B run under several connection counts.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/${1:-staged_conn}; mkdir -p $O
for rep in 1 2; do
  for c in 8 32 1 16 4; do
    CUDA_DEVICE_MAX_CONNECTIONS=$c timeout 120 python tools/staged_ab.py 16 3 | sed "s/}/, \"max_connections\": $c}/" >> $O/out.jsonl 2>>$O/err.log
  done
done
CUDA_DEVICE_MAX_CONNECTIONS=32 timeout 300 python tools/pipe_kernels_py.py > $O/pkp32.jsonl 2>&1
