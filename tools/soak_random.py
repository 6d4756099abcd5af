#!/usr/bin/env python
"""Randomised multi-threaded soak of the whole API (tests/ only cover fixed
mixes): T host threads, each on its own stream, loop for S seconds over random
(direction, mode, key size, page count, page size, residency, in place, host
path, single or mixed keys) batches; every output is compared byte for byte
with the oracle (test infrastructure, as in tests/).  Prints one JSON line.

usage: python tools/soak_random.py [seconds=600] [threads=4]"""
import json
import os
import sys
import threading
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_1305_3345_b200 as kg  # noqa: E402
import synth  # noqa: E402
from gpu_util import oracle_pages  # noqa: E402

KEY_IDS = [(10 + t, 40 + t) for t in range(16)]  # per thread: single-key slot, and mixed-key base


def main(seconds=600, threads=4):
    torch.cuda.init()
    kg.init(0)
    keys = {}
    for kb in (16, 24, 32):
        for j in range(4):
            kid = 100 + 10 * (kb // 8) + j
            keys[kid] = synth.make_key(kb, seed=kid)
            kg.set_key(kid, keys[kid])
    stop = time.time() + seconds
    stats = {"batches": 0, "bytes": 0, "mismatches": 0, "errors": []}
    lock = threading.Lock()

    def worker(tid):
        rng = np.random.default_rng(7000 + tid)
        s = torch.cuda.Stream()
        while time.time() < stop:
            try:
                d = int(rng.integers(0, 2))
                mode = int(rng.integers(0, 2))
                kb = int(rng.choice([16, 24, 32]))
                n = int(rng.choice([1, 2, 7, 33, 150, 300, 1200]))
                pb = 16 * int(rng.choice([1, 3, 16, 32, 64, 256]))
                where = str(rng.choice(["device", "pinned"]))
                inplace = bool(rng.integers(0, 2))
                mixed = bool(rng.integers(0, 3) == 0)
                seed = int(rng.integers(0, 1 << 30))
                data = synth.make_pages(n, pb, seed=seed)
                ivs = synth.make_ivs(n, seed=seed + 1) if mode == 0 else None
                kids = [100 + 10 * (kb // 8) + j for j in range(4)]
                if mixed:
                    ids = np.array(kids, dtype=np.uint16)[rng.integers(0, 4, n)]
                    exp = np.empty_like(data)
                    for p in range(n):
                        sl = slice(p * pb, (p + 1) * pb)
                        exp[sl] = oracle_pages(d, mode, keys[int(ids[p])], data[sl], 1, pb,
                                               None if ivs is None else ivs[16 * p:16 * p + 16])
                else:
                    kid = kids[int(rng.integers(0, 4))]
                    exp = oracle_pages(d, mode, keys[kid], data, n, pb, ivs)
                t_in = torch.from_numpy(data)
                t_in = t_in.cuda() if where == "device" else t_in.pin_memory()
                t_out = t_in if inplace else (torch.empty_like(t_in) if where == "device"
                                              else torch.empty_like(t_in).pin_memory())
                t_iv = None if ivs is None else (torch.from_numpy(ivs).cuda() if where == "device"
                                                 else torch.from_numpy(ivs).pin_memory())
                torch.cuda.synchronize()
                if mixed:
                    t_ids = torch.from_numpy(ids.astype(np.int16)).cuda()
                    t = kg.submit_pages_keyed(d, mode, t_in, t_out, n, pb, t_iv, t_ids, kb, s)
                else:
                    t = kg.submit_pages(d, mode, t_in, t_out, n, pb, t_iv, kid, s)
                kg.wait(t)
                s.synchronize()
                got = t_out.cpu().numpy()
                with lock:
                    stats["batches"] += 1
                    stats["bytes"] += n * pb
                    if not np.array_equal(got, exp):
                        stats["mismatches"] += 1
                        stats["errors"].append(dict(tid=tid, d=d, mode=mode, kb=kb, n=n, pb=pb, where=where,
                                                    inplace=inplace, mixed=mixed, seed=seed))
            except Exception as e:  # noqa: BLE001
                with lock:
                    stats["errors"].append(f"tid {tid}: {e!r}")
                    stats["mismatches"] += 1

    ths = [threading.Thread(target=worker, args=(t,)) for t in range(threads)]
    for th in ths:
        th.start()
    # a host-path switcher: the global host path changes under the workers' feet
    hp_rng = np.random.default_rng(1)
    while time.time() < stop:
        kg.set_host_path(int(hp_rng.integers(0, 3)), int(hp_rng.choice([1 << 16, 1 << 20, 32 << 20])))
        time.sleep(0.5)
    for th in ths:
        th.join()
    kg.set_host_path(kg.HOST_AUTO, 32 << 20)
    stats["errors"] = stats["errors"][:20]
    print(json.dumps({"test": "soak_random", "seconds": seconds, "threads": threads, **stats}), flush=True)
    return 1 if stats["mismatches"] else 0


if __name__ == "__main__":
    sys.exit(main(*(int(a) for a in sys.argv[1:])))
