#!/bin/bash
# The non-BASELINE workloads (row f1: ECB both ways, mixed keys; in place) on the final code
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/${1:-r2_modes}
mkdir -p $O
python bench.py --steps 20 --warmup 5 --no-sweep --no-cpu-baseline --extra ecb_dec,ecb_enc,c2_keyed,c3_keyed,c2_inplace,ecb_dec_inplace > $O/modes.json 2> $O/modes.err
python - <<'PY'
import json
l = [x for x in open("gpurun_out/r2_modes/modes.json") if x.startswith("{")][-1]
d = json.loads(l)
for k, v in [("c2", d)] + list(d["configs"].items()):
    e = v.get("e2e") or {}
    print(k, round(v["value"], 1), round(v["roofline"]["frac"], 4), v["check"]["mismatched_pages"], e.get("value") and round(e["value"], 2))
PY
