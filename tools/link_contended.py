#!/usr/bin/env python
"""Per-direction host-link rates while the other direction is busy the whole
time (the other copy is 2x longer), plus the equal-bytes duplex time
(bench_link.py's number), and the staged pipeline at several (chunk, slots)
settings through the library.  One JSON line per measurement."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def ev_pair():
    return torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def main(mib=256, reps=5):
    n = mib << 20
    h_src = torch.empty(2 * n, dtype=torch.uint8).pin_memory()
    h_dst = torch.empty(2 * n, dtype=torch.uint8).pin_memory()
    d_a = torch.empty(2 * n, dtype=torch.uint8, device="cuda")
    d_b = torch.empty(2 * n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def run(h2d_bytes, d2h_bytes):
        best = None
        for _ in range(reps):
            torch.cuda.synchronize()
            (a0, a1), (b0, b1) = ev_pair(), ev_pair()
            start = torch.cuda.Event()
            start.record()
            s1.wait_event(start)
            s2.wait_event(start)
            with torch.cuda.stream(s1):
                a0.record()
                if h2d_bytes:
                    d_a[:h2d_bytes].copy_(h_src[:h2d_bytes], non_blocking=True)
                a1.record()
            with torch.cuda.stream(s2):
                b0.record()
                if d2h_bytes:
                    h_dst[:d2h_bytes].copy_(d_b[:d2h_bytes], non_blocking=True)
                b1.record()
            torch.cuda.synchronize()
            r = (a0.elapsed_time(a1) / 1e3, b0.elapsed_time(b1) / 1e3)
            best = r if best is None else (min(best[0], r[0]), min(best[1], r[1]))
        return best

    th, _ = run(n, 0)
    _, td = run(0, n)
    print(json.dumps({"test": "solo", "h2d_gbs": n / th / 1e9, "d2h_gbs": n / td / 1e9}), flush=True)
    th, td = run(n, 2 * n)
    print(json.dumps({"test": "h2d_while_d2h_busy", "h2d_gbs": n / th / 1e9}), flush=True)
    th, td = run(2 * n, n)
    print(json.dumps({"test": "d2h_while_h2d_busy", "d2h_gbs": n / td / 1e9}), flush=True)
    th, td = run(n, n)
    print(json.dumps({"test": "equal_bytes_duplex", "h2d_s": th, "d2h_s": td,
                      "per_direction_gbs": n / max(th, td) / 1e9}), flush=True)

    # several streams per direction (several copy engines?)
    ss = [torch.cuda.Stream() for _ in range(8)]

    def multi(nh, nd, bh, bd):
        best = None
        for _ in range(reps):
            torch.cuda.synchronize()
            start = torch.cuda.Event(enable_timing=True)
            start.record()
            evs = []
            for k in range(nh):
                s = ss[k]
                s.wait_event(start)
                with torch.cuda.stream(s):
                    e0, e1 = ev_pair()
                    e0.record()
                    d_a[k * bh:(k + 1) * bh].copy_(h_src[k * bh:(k + 1) * bh], non_blocking=True)
                    e1.record()
                    evs.append(("h", e0, e1))
            for k in range(nd):
                s = ss[4 + k]
                s.wait_event(start)
                with torch.cuda.stream(s):
                    e0, e1 = ev_pair()
                    e0.record()
                    h_dst[k * bd:(k + 1) * bd].copy_(d_b[k * bd:(k + 1) * bd], non_blocking=True)
                    e1.record()
                    evs.append(("d", e0, e1))
            torch.cuda.synchronize()
            th = max([start.elapsed_time(e1) for kind, e0, e1 in evs if kind == "h"] or [0]) / 1e3
            td = max([start.elapsed_time(e1) for kind, e0, e1 in evs if kind == "d"] or [0]) / 1e3
            r = (th, td)
            best = r if best is None else (min(best[0], r[0]), min(best[1], r[1]))
        return best

    for nh in (1, 2, 4):
        th, _ = multi(nh, 0, n // nh, 0)
        print(json.dumps({"test": f"h2d_solo_{nh}streams", "h2d_gbs": n / th / 1e9}), flush=True)
        th, _ = multi(nh, 1, n // nh, 2 * n)
        print(json.dumps({"test": f"h2d_{nh}streams_while_d2h_busy", "h2d_gbs": n / th / 1e9}), flush=True)
        th, td = multi(nh, nh, n // nh, n // nh)
        print(json.dumps({"test": f"equal_bytes_duplex_{nh}+{nh}streams", "per_direction_gbs": n / max(th, td) / 1e9}),
              flush=True)

    # the staged pipeline through the library, 256 MiB AES-128-CBC decrypt, pinned in/out
    import numpy as np
    import paper_1305_3345_b200 as kg
    import synth
    kg.init(0)
    kg.set_key(0, synth.make_key(16))
    npg = n // 4096
    hx = torch.from_numpy(synth.make_pages(npg, 4096)).pin_memory()
    hiv = torch.from_numpy(synth.make_ivs(npg)).pin_memory()
    ho = torch.empty_like(hx).pin_memory()
    kg.set_host_path(kg.HOST_STAGED)
    for chunk_mib, slots in [(16, 3), (16, 8), (32, 8), (8, 8), (4, 8), (64, 4)]:
        kg.set_pipeline(chunk_mib << 20, slots)
        for _ in range(2):
            kg.wait(kg.submit_pages(1, 0, hx, ho, npg, 4096, hiv, 0))
        e0, e1 = ev_pair()
        torch.cuda.synchronize()
        e0.record()
        K = 10
        for _ in range(K):
            kg.wait(kg.submit_pages(1, 0, hx, ho, npg, 4096, hiv, 0))
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 1e3 / K
        print(json.dumps({"test": "staged_pipeline", "chunk_mib": chunk_mib, "slots": slots,
                          "gbs": n / t / 1e9}), flush=True)


if __name__ == "__main__":
    main(*(int(a) for a in sys.argv[1:]))
