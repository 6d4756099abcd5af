#!/usr/bin/env python
"""Scan the pinned-host staging pipeline (chunk bytes x slots) on the C2
batch (256 MiB AES-128-CBC decrypt, pinned in/out/IVs): e2e GB/s through
kg_submit_pages + kg_wait.  JSON line per setting."""
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
hx = torch.from_numpy(synth.make_pages(n, PB)).pin_memory()
hiv = torch.from_numpy(synth.make_ivs(n)).pin_memory()
hout = torch.empty_like(hx).pin_memory()
s = torch.cuda.current_stream()
for chunk_mib in (1, 2, 4, 8, 16, 32):
    for slots in (2, 3, 4, 6):
        kg.set_pipeline(chunk_mib << 20, slots)
        for _ in range(2):
            kg.wait(kg.submit_pages(1, 0, hx, hout, n, PB, hiv, 0, s))
        reps = 8
        t0 = time.perf_counter()
        for _ in range(reps):
            kg.wait(kg.submit_pages(1, 0, hx, hout, n, PB, hiv, 0, s))
        dt = (time.perf_counter() - t0) / reps
        print(json.dumps({"chunk_mib": chunk_mib, "slots": slots, "gbs": n * PB / dt / 1e9, "ms": dt * 1e3}), flush=True)
