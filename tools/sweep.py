#!/usr/bin/env python
"""BASELINE.json config 4: request batch-size sweep, 1 page .. 2^18 pages
(4 KiB .. 1 GiB), AES-128-CBC decrypt, 1 B200.  For each size: caller-
observed latency (submit -> kg_wait returns, wall clock) for HBM-resident
and pinned-host-resident batches (p10/p50/p90), GB/s, and the oracle's
latency on the host cores (1 thread and all threads) for sizes it finishes
quickly.  The GPU/CPU crossover is the smallest size where GPU latency <=
the better oracle latency (a tie counts for the GPU).
Writes JSON lines (one per size) and a summary line."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1305_3345_b200 as kg  # noqa: E402
import synth  # noqa: E402

PB = 4096


def pct(v, q):
    return float(np.percentile(np.array(v), q))


def lat(fn, reps):
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return ts


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kmax", type=int, default=18)
    ap.add_argument("--oracle-kmax", type=int, default=12)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    kg.init(0)
    key = synth.make_key(16)
    kg.set_key(0, key)
    threads = len(os.sched_getaffinity(0))
    nmax = 1 << a.kmax
    data = torch.from_numpy(synth.make_pages(nmax, PB))
    ivs = torch.from_numpy(synth.make_ivs(nmax))
    dx, div = data.cuda(), ivs.cuda()
    dout = torch.empty_like(dx)
    hx, hiv = data.pin_memory(), ivs.pin_memory()
    hout = torch.empty_like(hx).pin_memory()
    s = torch.cuda.current_stream()
    rows = []
    lines = []
    for k in range(a.kmax + 1):
        n = 1 << k
        reps = 200 if n * PB < (1 << 20) else (50 if n * PB < (64 << 20) else 10)

        def run_hbm():
            kg.wait(kg.submit_pages(1, 0, dx, dout, n, PB, div, 0, s))

        def run_pin():
            kg.wait(kg.submit_pages(1, 0, hx, hout, n, PB, hiv, 0, s))

        for f in (run_hbm, run_pin):
            for _ in range(3):
                f()
        th = lat(run_hbm, reps)
        kg.set_host_path(kg.HOST_STAGED)
        tp = lat(run_pin, reps)
        kg.set_host_path(kg.HOST_ZEROCOPY)
        tz = lat(run_pin, reps)
        kg.set_host_path(kg.HOST_AUTO, 32 << 20)
        tn = tnp = None
        if n <= 4096:  # the NSK (row f3), direct doorbell, 16 SMs
            kg.nsk_start(16, kg.NSK_DIRECT | kg.NSK_NOCAL, 5000)
            for _ in range(5):
                run_hbm()
            tn = lat(run_hbm, reps)
            tnp = lat(run_pin, reps)
            kg.nsk_stop()
        row = {"pages": n, "bytes": n * PB,
               "hbm_us_p10": 1e6 * pct(th, 10), "hbm_us_p50": 1e6 * pct(th, 50), "hbm_us_p90": 1e6 * pct(th, 90),
               "pinned_us_p10": 1e6 * pct(tp, 10), "pinned_us_p50": 1e6 * pct(tp, 50), "pinned_us_p90": 1e6 * pct(tp, 90)}
        row["zerocopy_us_p50"] = 1e6 * pct(tz, 50)
        if tn:
            row["nsk_hbm_us_p50"] = 1e6 * pct(tn, 50)
            row["nsk_pinned_us_p50"] = 1e6 * pct(tnp, 50)
        row["zerocopy_gbs"] = n * PB / (row["zerocopy_us_p50"] * 1e-6) / 1e9
        row["hbm_gbs"] = n * PB / (row["hbm_us_p50"] * 1e-6) / 1e9
        row["pinned_gbs"] = n * PB / (row["pinned_us_p50"] * 1e-6) / 1e9
        if k <= a.oracle_kmax:
            import oracle
            c = data[: n * PB].numpy()
            iv = ivs[: 16 * n].numpy()
            r1 = 20 if k < 6 else 3
            t1 = lat(lambda: oracle.pages(1, 0, key, c, n, PB, iv, threads=1), r1)
            tt = lat(lambda: oracle.pages(1, 0, key, c, n, PB, iv, threads=threads), r1)
            row["oracle_1t_us_p50"] = 1e6 * pct(t1, 50)
            row["oracle_all_us_p50"] = 1e6 * pct(tt, 50)
            row["oracle_best_us"] = min(row["oracle_1t_us_p50"], row["oracle_all_us_p50"])
        # context line, NOT the oracle: single-core OpenSSL (AES-NI) CBC, like the
        # paper's SSE-optimised in-kernel AES comparator
        try:
            from cryptography.hazmat.primitives.ciphers import Cipher, algorithms, modes
            cb = data[: n * PB].numpy().tobytes()
            ivb = ivs[: 16 * n].numpy().tobytes()

            def ossl():
                for p in range(n):
                    d = Cipher(algorithms.AES(key), modes.CBC(ivb[16 * p:16 * p + 16])).decryptor()
                    d.update(cb[p * PB:(p + 1) * PB])

            to = lat(ossl, 20 if k < 8 else 3)
            row["openssl_aesni_1core_us_p50"] = 1e6 * pct(to, 50)
        except Exception:  # noqa: BLE001
            pass
        rows.append(row)
        lines.append(json.dumps(row))
        print(lines[-1], flush=True)
    summ = {"summary": "c4_sweep", "oracle_threads": threads}
    for res in ("hbm", "pinned", "zerocopy", "nsk_hbm", "nsk_pinned"):
        for ref, key_ in (("oracle", "oracle_best_us"), ("openssl_aesni_1core", "openssl_aesni_1core_us_p50")):
            cross = None
            for r in rows:
                if key_ in r and f"{res}_us_p50" in r and r[f"{res}_us_p50"] <= r[key_]:
                    cross = r["bytes"]
                    break
            summ[f"crossover_bytes_{res}_vs_{ref}"] = cross
    print(json.dumps(summ), flush=True)
    if a.out:
        with open(a.out, "w") as f:
            f.write("\n".join(lines + [json.dumps(summ)]) + "\n")


if __name__ == "__main__":
    main()
