"""The N>1 host logic on CPU: two gloo ranks on 127.0.0.1 shard a batch by
contiguous page range (synth.shard), process their shards independently (the
oracle stands in for the device here -- no data-path collective exists), and
the MAX/SUM scalar reductions bench.py uses give the whole-job figures."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, pb, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    lo, hi = synth.shard(n, rank, world)
    key = synth.make_key(16)
    data = synth.make_pages(hi - lo, pb, first_page=lo)
    ivs = synth.make_ivs(hi - lo, first_page=lo)
    out = oracle.pages(0, 0, key, data, hi - lo, pb, ivs)
    # bench.py's reductions: MAX of elapsed, SUM of mismatches / pages
    t = torch.tensor([0.25 * (rank + 1), float(hi - lo)], dtype=torch.float64)
    tmax = t.clone()
    dist.all_reduce(tmax[:1], op=dist.ReduceOp.MAX)
    tsum = t.clone()
    dist.all_reduce(tsum[1:], op=dist.ReduceOp.SUM)
    gathered = [None] * world
    dist.all_gather_object(gathered, (lo, hi, out.tobytes()))
    if rank == 0:
        q.put((float(tmax[0]), float(tsum[1]), gathered))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_page_range_sharding():
    n, pb, world = 37, 512, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, pb, q)) for r in range(world)]
    for p in procs:
        p.start()
    tmax, pages, gathered = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert tmax == 0.5 and pages == n
    import oracle
    full = oracle.pages(0, 0, synth.make_key(16), synth.make_pages(n, pb), n, pb, synth.make_ivs(n))
    parts = sorted(gathered)
    assert parts[0][0] == 0 and parts[-1][1] == n
    joined = b"".join(p[2] for p in parts)
    assert np.array_equal(np.frombuffer(joined, dtype=np.uint8), full)
