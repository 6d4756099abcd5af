#!/usr/bin/env python
"""C5 pinned-host e2e, step by step: one 64 GiB AES-128-CBC decrypt batch in
place in kg_alloc_pinned host memory, submitted and waited S times; prints one
JSON line per step (ms, GB/s) plus the NUMA placement of the buffer
(/proc/self/numa_maps) and the host's free memory per node.  Diagnoses the
spread of bench.py's C5 e2e steps (profiles/r2_e2e).

usage: python tools/c5_e2e_steps.py [steps=8] [gib=64]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1305_3345_b200 as kg  # noqa: E402
import synth  # noqa: E402

PB = 4096


def numa_of(addr):
    """Pages per NUMA node of the mapping that contains addr (numa_maps N<node>=<pages>)."""
    best = None
    try:
        with open("/proc/self/numa_maps") as f:
            for line in f:
                parts = line.split()
                start = int(parts[0], 16)
                if start <= addr and (best is None or start > best[0]):
                    fields = dict(kv.split("=", 1) for kv in parts[2:] if "=" in kv)
                    nodes = {k: int(v) for k, v in fields.items() if k[:1] == "N" and k[1:].isdigit()}
                    best = (start, nodes, fields.get("kernelpagesize_kB"))
    except Exception as e:  # noqa: BLE001
        return {"error": str(e)}
    return None if best is None else {"start": hex(best[0]), "pages_per_node": best[1], "page_kB": best[2]}


def main(steps=8, gib=64):
    n = gib * (1 << 30) // PB
    torch.cuda.set_device(0)
    kg.init(0)
    kg.set_key(0, synth.make_key(16))
    t0 = time.perf_counter()
    hx = kg.alloc_pinned(n * PB)
    hiv = kg.alloc_pinned(16 * n)
    t_alloc = time.perf_counter() - t0
    M = 65537
    pat = torch.from_numpy(synth.make_pages(M, PB)).view(M, PB)
    hv = hx.view(n, PB)
    for s in range(0, n, M):
        e = min(n, s + M)
        hv[s:e].copy_(pat[:e - s])
    hiv.view(n, 16)[:] = torch.from_numpy(synth.make_ivs(1)).view(1, 16)
    print(json.dumps({"alloc_s": round(t_alloc, 2), "numa": numa_of(hx.data_ptr())}), flush=True)
    try:
        with open("/sys/devices/system/node/node0/meminfo") as f:
            print(json.dumps({"node0": [l.strip() for l in f if "MemFree" in l or "MemTotal" in l]}), flush=True)
        with open("/sys/devices/system/node/node1/meminfo") as f:
            print(json.dumps({"node1": [l.strip() for l in f if "MemFree" in l or "MemTotal" in l]}), flush=True)
    except OSError:
        pass
    for i in range(steps):
        t = time.perf_counter()
        kg.wait(kg.submit_pages(1, 0, hx, hx, n, PB, hiv, 0))  # decrypt in place, as bench.py's C5 e2e
        dt = time.perf_counter() - t
        print(json.dumps({"step": i, "ms": round(1e3 * dt, 1),
                          "gbs": round(n * PB / dt / 1e9, 2)}), flush=True)
    kg.free_pinned(hx)
    kg.free_pinned(hiv)


if __name__ == "__main__":
    main(*(int(a) for a in sys.argv[1:]))
