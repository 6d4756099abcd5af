#!/bin/bash
# A/B: byte-3 T-table offsets on the FMA pipe (IMAD.HI + IMAD) instead of PRMT (KG_T3_FMA; ALU pipe relief)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/${1:-r2_t3fma}
mkdir -p $O
for rep in 1 2; do
for v in product t3fma; do
  L=$PWD/paper_1305_3345_b200/libkgpu.so; [ $v != product ] && L=$PWD/build/ab/$v/libkgpu.so
  KG_LIBKGPU=$L python bench.py --steps 20 --warmup 5 --no-e2e --no-sweep --no-cpu-baseline --extra c3,c4_1gib,ecb_dec > $O/${v}_r$rep.json 2> $O/${v}_r$rep.err
done
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/r2_t3fma/*.json")):
    l = [x for x in open(f) if x.startswith("{")]
    if not l: print(f, "no line"); continue
    d = json.loads(l[-1])
    print(f.split("/")[-1], round(d["value"], 1), {k: round(v["value"], 1) for k, v in d["configs"].items()},
          d["check"]["mismatched_pages"], [v["check"]["mismatched_pages"] for v in d["configs"].values()])
PY
