#!/bin/bash
# Round-2 code under the sanitizers: compute-sanitizer (memcheck, racecheck,
# synccheck, initcheck) over tools/sanitize_run.py (every kernel family, staged
# warm/cold batches, keyed batches, the NSK), the ThreadSanitizer build of the
# runtime (build/soak_tsan), and the randomised oracle-checked API soak.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/${1:-r2_sanitize}
mkdir -p $O
for t in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_run.py > $O/$t.log 2>&1
  echo "rc=$?" >> $O/$t.log
done
TSAN_OPTIONS="halt_on_error=0 report_signal_unsafe=0" timeout 900 ./build/soak_tsan > $O/soak_tsan.log 2>&1
echo "rc=$?" >> $O/soak_tsan.log
timeout 600 python tools/soak_random.py ${SOAK_S:-300} 4 > $O/soak_random.json 2>&1
echo "rc=$?" >> $O/soak_random.json
for f in $O/*.log $O/*.json; do echo "== $f"; tail -3 $f; done
