#!/usr/bin/env python
"""Host-link copy bandwidth (the pinned-host roofline):
pinned cudaMemcpyAsync H2D alone, D2H alone, and both concurrently on two
streams, 256 MiB, best of N, CUDA-event timed.  One JSON line."""
import json
import sys

import torch


def main(mib=256, reps=10):
    n = mib << 20
    h_src = torch.empty(n, dtype=torch.uint8).pin_memory()
    h_dst = torch.empty(n, dtype=torch.uint8).pin_memory()
    d_a = torch.empty(n, dtype=torch.uint8, device="cuda")
    d_b = torch.empty(n, dtype=torch.uint8, device="cuda")
    h_src.fill_(7)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(fn):
        best = 1e9
        for _ in range(reps):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            for s in (s1, s2):
                torch.cuda.current_stream().wait_stream(s)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) / 1e3)
        return best

    def h2d():
        with torch.cuda.stream(s1):
            d_a.copy_(h_src, non_blocking=True)

    def d2h():
        with torch.cuda.stream(s2):
            h_dst.copy_(d_b, non_blocking=True)

    def both():
        h2d()
        d2h()

    t_h2d, t_d2h, t_both = timed(h2d), timed(d2h), timed(both)
    out = {"test": "host_link", "bytes": n, "h2d_gbs": n / t_h2d / 1e9, "d2h_gbs": n / t_d2h / 1e9,
           "duplex_h2d_plus_d2h_gbs": 2 * n / t_both / 1e9, "duplex_per_direction_gbs": n / t_both / 1e9,
           "device": torch.cuda.get_device_name()}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main(*(int(a) for a in sys.argv[1:]))
