#!/bin/bash
# A/B: compact inverse S-box (KG_SI_COMPACT: 32 KiB instead of a 64 KiB region, more L1 for the
# texture cache) x blocks per lane (KG_GROUP 2 / 4), decrypt configs through bench.py; parity of c1g2
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/${1:-r2_si_group}
mkdir -p $O
for rep in 1 2; do
for v in product c1g2 c1g4 c0g4; do
  L=$PWD/paper_1305_3345_b200/libkgpu.so; [ $v != product ] && L=$PWD/build/ab/$v/libkgpu.so
  KG_LIBKGPU=$L python bench.py --steps 20 --warmup 5 --no-e2e --no-sweep --no-cpu-baseline --extra c4_1gib,ecb_dec > $O/${v}_r$rep.json 2> $O/${v}_r$rep.err
done
done
KG_LIBKGPU=$PWD/build/ab/c1g2/libkgpu.so timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_keyed_gpu.py tests/test_fullsize_gpu.py tests/test_align_gpu.py -q -x -p no:cacheprovider > $O/pytest_c1g2.txt 2>&1; echo rc=$? >> $O/pytest_c1g2.txt
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/r2_si_group/*.json")):
    l = [x for x in open(f) if x.startswith("{")]
    if not l: print(f, "no line"); continue
    d = json.loads(l[-1])
    print(f.split("/")[-1], round(d["value"], 1), {k: round(v["value"], 1) for k, v in d["configs"].items()},
          d["check"]["mismatched_pages"], [v["check"]["mismatched_pages"] for v in d["configs"].values()])
PY
tail -n 2 $O/pytest_c1g2.txt
