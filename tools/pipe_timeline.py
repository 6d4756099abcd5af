#!/usr/bin/env python
"""Per-chunk start/end events of every stage of the torch-stream staged
pipeline (H2D, compute, D2H) for compute = none / aes: when does each copy
actually start, and how long does it run?"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1305_3345_b200 as kg  # noqa: E402
import synth  # noqa: E402


def ev(stream):
    e = torch.cuda.Event(enable_timing=True)
    e.record(stream)
    return e


def main():
    PB, total, chunk, slots = 4096, 256 << 20, 16 << 20, 3
    n, cp = total // PB, chunk // PB
    kg.init(0)
    kg.set_key(0, synth.make_key(16))
    hx = torch.from_numpy(synth.make_pages(n, PB)).pin_memory()
    ho = torch.empty_like(hx).pin_memory()
    div = torch.from_numpy(synth.make_ivs(n)).cuda()
    slot_in = [torch.empty(chunk, dtype=torch.uint8, device="cuda") for _ in range(slots)]
    slot_out = [torch.empty(chunk, dtype=torch.uint8, device="cuda") for _ in range(slots)]
    sh, sk, sd = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    nch = total // chunk
    for kind in ["none", "aes", "none", "aes"]:
        torch.cuda.synchronize()
        t0 = ev(torch.cuda.current_stream())
        for s_ in (sh, sk, sd):
            s_.wait_event(t0)
        freed = [None] * slots
        rec = []
        tickets = []
        for i in range(nch):
            s = i % slots
            r = {}
            if freed[s] is not None:
                sh.wait_event(freed[s])
            r["hs"] = ev(sh)
            with torch.cuda.stream(sh):
                slot_in[s].copy_(hx[i * chunk:(i + 1) * chunk], non_blocking=True)
            r["he"] = ev(sh)
            sk.wait_event(r["he"])
            r["ks"] = ev(sk)
            src = slot_in[s]
            if kind == "aes":
                tickets.append(kg.submit_pages(1, 0, slot_in[s], slot_out[s], cp, PB,
                                               div[16 * i * cp:16 * (i + 1) * cp], 0, sk))
                src = slot_out[s]
            r["ke"] = ev(sk)
            sd.wait_event(r["ke"])
            r["ds"] = ev(sd)
            with torch.cuda.stream(sd):
                ho[i * chunk:(i + 1) * chunk].copy_(src, non_blocking=True)
            r["de"] = ev(sd)
            freed[s] = r["de"]
            rec.append(r)
        torch.cuda.synchronize()
        for tk in tickets:
            kg.wait(tk)
        out = [{k: round(t0.elapsed_time(v) * 1e3, 1) for k, v in r.items()} for r in rec]
        tot = out[-1]["de"]
        print(json.dumps({"test": "pipe_timeline", "compute": kind, "total_us": tot, "gbs": total / tot / 1e3,
                          "chunks": out}), flush=True)


if __name__ == "__main__":
    main()
