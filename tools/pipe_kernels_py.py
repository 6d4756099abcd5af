#!/usr/bin/env python
"""The staged pipeline rebuilt from torch streams/events around different
compute steps per 16 MiB chunk (pinned in -> device slot -> pinned out),
to see how much the compute kernel itself slows the copy engines:
none, a light torch kernel, and the AES kernel through kg_submit_pages on
device memory.  256 MiB, 3 slots."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1305_3345_b200 as kg  # noqa: E402
import synth  # noqa: E402


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
    def h2d(i, freed, loaded):
        s = i % slots
        with torch.cuda.stream(sh):
            if freed[s] is not None:
                sh.wait_event(freed[s])
            slot_in[s].copy_(hx[i * chunk:(i + 1) * chunk], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(sh)
            loaded[i] = ev

    nch = total // chunk
    for kind, la in [("none", 0), ("torch_add", 0), ("aes", 0), ("aes", 1), ("aes", 2), ("torch_add", 1),
                     ("none", 1)]:
        best = 0
        for rep in range(4):
            torch.cuda.synchronize()
            freed = [None] * slots
            loaded = [None] * nch
            t0 = time.perf_counter()
            tickets = []
            # issue order: the H2D of chunk i+la is enqueued before the D2H of chunk i
            for i in range(min(la, nch)):
                h2d(i, freed, loaded)
            for i in range(nch):
                if i + la < nch:
                    h2d(i + la, freed, loaded)
                s = i % slots
                src = slot_in[s]
                with torch.cuda.stream(sk):
                    sk.wait_event(loaded[i])
                    if kind == "torch_add":
                        slot_out[s].copy_(slot_in[s])
                        src = slot_out[s]
                    elif kind == "aes":
                        tickets.append(kg.submit_pages(1, 0, slot_in[s], slot_out[s], cp, PB,
                                                       div[16 * i * cp:16 * (i + 1) * cp], 0, sk))
                        src = slot_out[s]
                    done = torch.cuda.Event()
                    done.record(sk)
                with torch.cuda.stream(sd):
                    sd.wait_event(done)
                    ho[i * chunk:(i + 1) * chunk].copy_(src, non_blocking=True)
                    fr = torch.cuda.Event()
                    fr.record(sd)
                    freed[s] = fr
            torch.cuda.synchronize()
            t = time.perf_counter() - t0
            for tk in tickets:
                kg.wait(tk)
            best = max(best, total / t / 1e9)
        print(json.dumps({"test": "pipe_kernels_py", "compute": kind, "h2d_lookahead": la, "gbs": best}), flush=True)

if __name__ == "__main__":
    main()
