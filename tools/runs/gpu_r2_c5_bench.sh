#!/bin/bash
# C5 through bench.py (2 warm-up + 4 timed e2e steps, per-step times in the line), twice; then the default line
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/${1:-r2_c5_bench}
mkdir -p $O
for rep in 1 2; do
python bench.py --workload c5 --extra none --steps 3 --warmup 3 --no-sweep --no-cpu-baseline > $O/c5_r$rep.json 2> $O/c5_r$rep.err
done
S0=$SECONDS; python3 bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "bench rc=$? wall_s=$((SECONDS - S0))" >> $O/bench.err
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/r2_c5_bench/*.json")):
    l = [x for x in open(f) if x.startswith("{")]
    if not l: print(f, "no line"); continue
    d = json.loads(l[-1])
    cs = [("head", d)] + list(d.get("configs", {}).items())
    for k, v in cs:
        e = v.get("e2e") or {}
        print(f, k, round(v["value"], 1), e.get("value") and round(e["value"], 2), e.get("link_frac") and round(e["link_frac"], 3), e.get("step_ms"))
PY
tail -n 1 $O/bench.err
