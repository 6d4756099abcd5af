#!/usr/bin/env python
"""Locate the GPU-vs-CPU latency crossover (BASELINE.json C4; PAPER.md:460-463
"8KB or larger") in a tools/sweep.py output: for each GPU path (launch on HBM
data, staged pinned, zero-copy pinned, NSK on HBM / pinned data) and each CPU
reference (the oracle on 1 thread / all threads, single-core OpenSSL AES-NI as
context), the smallest batch from which the GPU path's p50 latency is <= the
CPU's.  usage: python tools/crossover.py SWEEP.jsonl [--out FILE.json]"""
import argparse
import json


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("sweep")
    ap.add_argument("--out")
    a = ap.parse_args()
    rows = [json.loads(l) for l in open(a.sweep) if l.strip().startswith("{")]
    rows = [r for r in rows if "pages" in r]
    gpu = {"launch_hbm": "hbm_us_p50", "staged_pinned": "pinned_us_p50", "zerocopy_pinned": "zerocopy_us_p50",
           "nsk_hbm": "nsk_hbm_us_p50", "nsk_pinned": "nsk_pinned_us_p50"}
    cpu = {"oracle_1_thread": "oracle_1t_us_p50", "oracle_all_threads": "oracle_all_us_p50",
           "openssl_aesni_1_core (context)": "openssl_aesni_1core_us_p50"}
    out = {"source": a.sweep, "unit": "bytes (4 KiB pages)", "crossover": {}}
    for gname, gk in gpu.items():
        for cname, ck in cpu.items():
            pts = [r for r in rows if gk in r and ck in r]
            if not pts:
                continue
            first = None
            for r in pts:  # smallest size from which the GPU stays at or below the CPU
                if all(q[gk] <= q[ck] for q in pts if q["bytes"] >= r["bytes"]):
                    first = r["bytes"]
                    break
            out["crossover"][f"{gname} vs {cname}"] = {
                "bytes": first, "measured_range": [pts[0]["bytes"], pts[-1]["bytes"]],
                "note": None if first is not None else "GPU slower over the whole measured range"}
    s = json.dumps(out, indent=1)
    if a.out:
        open(a.out, "w").write(s + "\n")
    print(s)


if __name__ == "__main__":
    main()
