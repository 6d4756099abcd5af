#!/usr/bin/env python
"""Scan the pinned-host paths on the C2 batch (256 MiB AES-128-CBC decrypt,
pinned in/out/IVs): staged pipeline (chunk bytes x slots) and zero-copy;
e2e GB/s through kg_submit_pages + kg_wait, plus the host-side submit time
(request-queue enqueue cost).  JSON line per setting."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1305_3345_b200 as kg  # noqa: E402
import synth  # noqa: E402

PB = 4096
n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
kg.init(0)
kg.set_key(0, synth.make_key(16))
kg.set_key(1, synth.make_key(32))
hx = torch.from_numpy(synth.make_pages(n, PB)).pin_memory()
hiv = torch.from_numpy(synth.make_ivs(n)).pin_memory()
hout = torch.empty_like(hx).pin_memory()
s = torch.cuda.current_stream()


def run(label, direction=1, key_id=0, reps=8, **kw):
    for _ in range(2):
        kg.wait(kg.submit_pages(direction, 0, hx, hout, n, PB, hiv, key_id, s))
    tsub, ttot = 0.0, 0.0
    for _ in range(reps):
        t0 = time.perf_counter()
        t = kg.submit_pages(direction, 0, hx, hout, n, PB, hiv, key_id, s)
        t1 = time.perf_counter()
        kg.wait(t)
        t2 = time.perf_counter()
        tsub += t1 - t0
        ttot += t2 - t0
    print(json.dumps(dict(label=label, gbs=n * PB * reps / ttot / 1e9, ms=1e3 * ttot / reps,
                          submit_ms=1e3 * tsub / reps, **kw)), flush=True)


kg.set_host_path(kg.HOST_ZEROCOPY)
run("zerocopy_dec128")
run("zerocopy_enc256", direction=0, key_id=1)
kg.set_host_path(kg.HOST_STAGED)
run("staged_enc256_8MiB", direction=0, key_id=1)
for chunk_mib in (1, 2, 4, 8, 16, 32):
    for slots in (3, 4):
        kg.set_pipeline(chunk_mib << 20, slots)
        run("staged_dec128", chunk_mib=chunk_mib, slots=slots)
