#!/usr/bin/env python
"""CBC-encrypt chain kernel: GB/s of 1 GiB AES-256 batches at several page
sizes, for one KG_CHAIN_ALIGN value (set in the environment; read at kg_init).
One JSON line per page size.  profiles/r2_chain_align."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1305_3345_b200 as kg  # noqa: E402

torch.cuda.set_device(0)
kg.init(0)
kg.set_key(0, bytes(range(32)))
total = 1 << 30
x = torch.randint(0, 256, (total,), dtype=torch.uint8, device="cuda")
out = torch.empty_like(x)
for pb in [int(v) for v in (sys.argv[1:] or ["1024", "4096", "8192", "16384", "65536"])]:
    n = total // pb
    ivs = torch.zeros(16 * n, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        kg.wait(kg.submit_pages(kg.ENCRYPT, kg.MODE_CBC, x, out, n, pb, ivs, 0))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    ts = [kg.submit_pages(kg.ENCRYPT, kg.MODE_CBC, x, out, n, pb, ivs, 0) for _ in range(10)]
    e1.record()
    for t in ts:
        kg.wait(t)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(json.dumps({"page_bytes": pb, "n_pages": n, "chain_align": os.environ.get("KG_CHAIN_ALIGN", "default"),
                      "ms": round(ms, 4), "gbs": round(total / ms / 1e6, 2)}), flush=True)
