#!/usr/bin/env python
"""KG_TRACE timeline of C2 pinned-host batches (256 MiB AES-128-CBC decrypt,
kg_alloc_pinned in/out/IVs): per-chunk H2D / kernel / D2H completion times
(us) of the 3rd of 4 back-to-back batches, and the batch time.  Run with
KG_TRACE=1; the timeline is printed by the library on stderr at kg_wait."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1305_3345_b200 as kg  # noqa: E402
import synth  # noqa: E402

PB, n = 4096, 65536
torch.cuda.set_device(0)
kg.init(0)
kg.set_key(0, synth.make_key(16))
hx, hout, hiv = kg.alloc_pinned(n * PB), kg.alloc_pinned(n * PB), kg.alloc_pinned(16 * n)
hx.copy_(torch.from_numpy(synth.make_pages(n, PB)))
hiv.copy_(torch.from_numpy(synth.make_ivs(n)))
for i in range(4):
    t0 = time.perf_counter()
    kg.wait(kg.submit_pages(1, 0, hx, hout, n, PB, hiv, 0))
    print(f"batch {i}: {1e3 * (time.perf_counter() - t0):.3f} ms", file=sys.stderr, flush=True)
