#!/usr/bin/env python
"""Pinned H2D + D2H copy rates (256 MiB each way, concurrently) while another
stream keeps the SMs busy with (a) nothing, (b) the AES decrypt kernel on
unrelated device data, (c) a torch device-to-device copy kernel."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1305_3345_b200 as kg  # noqa: E402
import synth  # noqa: E402


def main():
    n = 256 << 20
    kg.init(0)
    kg.set_key(0, synth.make_key(16))
    h_src = torch.empty(n, dtype=torch.uint8).pin_memory()
    h_dst = torch.empty(n, dtype=torch.uint8).pin_memory()
    d_a = torch.empty(n, dtype=torch.uint8, device="cuda")
    d_b = torch.empty(n, dtype=torch.uint8, device="cuda")
    npg = (1 << 30) // 4096
    bx = torch.from_numpy(synth.make_pages(npg, 4096)).cuda()
    bo = torch.empty_like(bx)
    biv = torch.from_numpy(synth.make_ivs(npg)).cuda()
    s1, s2, s3 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    for load in ["none", "aes", "torch_copy", "none", "aes", "torch_copy"]:
        torch.cuda.synchronize()
        # background load: ~25 ms of work queued on s3
        tickets = []
        with torch.cuda.stream(s3):
            for _ in range(20):
                if load == "aes":
                    tickets.append(kg.submit_pages(1, 0, bx, bo, npg, 4096, biv, 0, s3))   # ~1.3 ms each
                elif load == "torch_copy":
                    for _ in range(3):
                        bo.copy_(bx)                                                   # ~0.4 ms each
        (a0, a1), (b0, b1) = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                              for _ in range(2)]
        with torch.cuda.stream(s1):
            a0.record()
            d_a.copy_(h_src, non_blocking=True)
            a1.record()
        with torch.cuda.stream(s2):
            b0.record()
            h_dst.copy_(d_b, non_blocking=True)
            b1.record()
        torch.cuda.synchronize()
        for t in tickets:
            kg.wait(t)
        print(json.dumps({"test": "copy_under_load", "load": load,
                          "h2d_gbs": n / (a0.elapsed_time(a1) / 1e3) / 1e9,
                          "d2h_gbs": n / (b0.elapsed_time(b1) / 1e3) / 1e9}), flush=True)


if __name__ == "__main__":
    main()
