#!/bin/bash
# compute-sanitizer over the small-config workload (one tool per pass).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/${1:-sanitize}
mkdir -p $O
for t in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_run.py > $O/$t.log 2>&1
  echo "rc=$?" >> $O/$t.log
done
