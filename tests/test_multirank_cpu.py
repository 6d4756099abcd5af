"""The N>1 host logic of bench.py on CPU, with bench.py's OWN code: two gloo
ranks on 127.0.0.1 take their shares with bench.plan (weak: a full batch per
rank; strong/C5: contiguous page ranges that partition the job), reduce with
bench.reduce_max / bench.reduce_sum, and report bench.job_bytes.  The sharded
oracle result of a small strong-scaling workload planned by bench.plan equals
the unsharded one (pages are independent: no data-path collective exists).
Plus bench.py's launcher: --gpus 2 without WORLD_SIZE re-launches itself as 2
ranks; a WORLD_SIZE that contradicts --gpus is refused."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT

import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


TINY = (37, 16, 0, 0, False, "strong", "tiny strong-scaling workload (test only)")


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sys.path.insert(0, ROOT)
    import bench
    import oracle
    bench.WORKLOADS["tiny"] = TINY
    res = {}
    for w in ("c2", "c3", "c5", "tiny"):
        res[w] = bench.plan(w, rank, world)
    # the reductions bench.py applies to per-rank timings and check counters
    tmax = bench.reduce_max(dist, [0.25 * (rank + 1), 10.0 - rank], "cpu")
    tsum = bench.reduce_sum(dist, [rank, 1.0], "cpu")
    # sharded work on the tiny strong workload, planned by bench.plan
    lo, n, _ = res["tiny"]
    pb = 512
    key = synth.make_key(16)
    out = oracle.pages(0, 0, key, synth.make_pages(n, pb, first_page=lo), n, pb, synth.make_ivs(n, first_page=lo))
    gathered = [None] * world
    dist.all_gather_object(gathered, (rank, res, out.tobytes()))
    if rank == 0:
        q.put((tmax, tsum, gathered, bench.job_bytes("c2", world, 3), bench.job_bytes("c5", world, 3)))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_plan_reductions_and_sharded_result():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    tmax, tsum, gathered, c2_bytes, c5_bytes = q.get(timeout=180)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert tmax == [0.5, 10.0] and tsum == [1.0, 2.0]
    plans = {r: res for r, res, _ in gathered}
    # weak: every rank its own full batch, disjoint page streams
    for w, n in (("c2", 65536), ("c3", 262144)):
        assert [plans[r][w] for r in range(world)] == [(0, n, "weak"), (n, n, "weak")]
    # strong (C5): contiguous ranges partitioning 2^24 pages
    c5 = [plans[r]["c5"] for r in range(world)]
    assert c5[0][0] == 0 and c5[0][0] + c5[0][1] == c5[1][0] and c5[1][0] + c5[1][1] == 16777216
    assert all(s == "strong" for _, _, s in c5)
    assert c2_bytes == 2 * 65536 * 4096 * 3          # weak: grows with W
    assert c5_bytes == 16777216 * 4096 * 3            # strong: fixed job
    # sharded == unsharded on the tiny strong workload
    import oracle
    n, pb = TINY[0], 512
    full = oracle.pages(0, 0, synth.make_key(16), synth.make_pages(n, pb), n, pb, synth.make_ivs(n))
    joined = b"".join(blob for _, _, blob in sorted(gathered))
    assert np.array_equal(np.frombuffer(joined, dtype=np.uint8), full)


def _bench(args, env_extra=None, timeout=240):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["PYTHONPATH"] = ROOT
    env.update(env_extra or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                          timeout=timeout, env=env)


def test_bench_self_launches_n_ranks(monkeypatch):
    """--gpus N without a launcher: bench.main re-runs bench.py under
    torch.distributed.run with N ranks on 127.0.0.1 and the same arguments
    (the real two-rank launch runs in tests/test_bench_gpu.py)."""
    sys.path.insert(0, ROOT)
    import bench
    calls = []
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(bench.subprocess, "call", lambda cmd, env=None: calls.append((cmd, env)) or 0)
    assert bench.main(["--gpus", "4", "--steps", "7", "--warmup", "3"]) == 0
    (cmd, env), = calls
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--master-addr=127.0.0.1" in cmd and "--nnodes=1" in cmd
    assert cmd[-7:] == [os.path.join(ROOT, "bench.py"), "--gpus", "4", "--steps", "7", "--warmup", "3"]
    assert env["NCCL_DEBUG"] == "INFO"
    calls.clear()
    monkeypatch.setenv("WORLD_SIZE", "4")       # already under a launcher: no re-launch
    monkeypatch.setattr(bench, "run_ours", lambda a: 0)
    assert bench.main(["--gpus", "4"]) == 0 and not calls


def test_bench_refuses_world_mismatch():
    r = _bench(["--gpus", "2"], {"WORLD_SIZE": "3", "RANK": "0"})
    assert r.returncode == 2
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert "refusing" in d["error"] and d["world"] == 3
