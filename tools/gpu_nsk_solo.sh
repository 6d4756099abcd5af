#!/bin/bash
# (historical: the KG_NSK_SOLO fast path was reverted after this A/B; profiles/r1_nsk/README.md)
# NSK solo fast path: tests + latency A/B (KG_NSK_SOLO).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/${1:-nsk_solo}; mkdir -p $O
timeout 900 python -m pytest tests/test_nsk_gpu.py -x -q > $O/pytest_nsk.log 2>&1; echo "rc=$?" >> $O/pytest_nsk.log
KG_NSK_SOLO=0 timeout 900 python -m pytest tests/test_nsk_gpu.py -x -q > $O/pytest_nsk_solo0.log 2>&1; echo "rc=$?" >> $O/pytest_nsk_solo0.log
for s in 1 0; do
  KG_NSK_SOLO=$s timeout 300 ./build/latency 2000 > $O/latency_solo$s.jsonl 2>&1; echo "rc=$?" >> $O/latency_solo$s.jsonl
done
