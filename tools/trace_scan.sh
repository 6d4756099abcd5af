#!/bin/bash
# Per-chunk timelines (KG_TRACE) of the staged pipeline, 256 MiB decrypt, under a few settings.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/${1:-trace_scan}; mkdir -p $O
KG_TRACE=1 timeout 120 python tools/trace_run.py 65536 16 > $O/t16_pdl.log 2>&1
KG_TRACE=1 KG_PDL=0 timeout 120 python tools/trace_run.py 65536 16 > $O/t16_nopdl.log 2>&1
KG_TRACE=1 timeout 120 python tools/trace_run.py 65536 32 > $O/t32.log 2>&1
