#!/usr/bin/env python
"""A/B of the staged pinned pipeline (256 MiB AES-128-CBC decrypt, pinned in/out):
one setting per process (KG_PDL is read once), K timed batches, GB/s."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1305_3345_b200 as kg  # noqa: E402
import synth  # noqa: E402


def main(chunk_mib=16, slots=3, k=10, direction=1, key_bytes=16, mib=256):
    n = (mib << 20) // 4096
    kg.init(0)
    kg.set_key(0, synth.make_key(key_bytes))
    hx = torch.from_numpy(synth.make_pages(n, 4096)).pin_memory()
    hiv = torch.from_numpy(synth.make_ivs(n)).pin_memory()
    ho = torch.empty_like(hx).pin_memory()
    kg.set_host_path(kg.HOST_STAGED)
    kg.set_pipeline(chunk_mib << 20, slots)
    for _ in range(3):
        kg.wait(kg.submit_pages(direction, 0, hx, ho, n, 4096, hiv, 0))
    torch.cuda.synchronize()
    steps = []
    t0 = time.perf_counter()
    for _ in range(k):
        ts = time.perf_counter()
        kg.wait(kg.submit_pages(direction, 0, hx, ho, n, 4096, hiv, 0))
        steps.append(round((time.perf_counter() - ts) * 1e3, 3))
    t = (time.perf_counter() - t0) / k
    print(json.dumps({"test": "staged_ab", "pdl": os.environ.get("KG_PDL", "1"), "chunk_mib": chunk_mib,
                      "slots": slots, "dir": direction, "key_bytes": key_bytes, "mib": mib,
                      "gbs": n * 4096 / t / 1e9, "step_ms": steps}), flush=True)


if __name__ == "__main__":
    main(*(int(a) for a in sys.argv[1:]))
