"""Row f3: the Non-Stop Kernel (persistent service kernel).
NB: while the NSK runs, DEVICE-wide synchronisation (torch.cuda.synchronize,
cudaDeviceSynchronize) waits for the persistent kernel's idle exit, so these
tests synchronise streams only.
Parity with the oracle through the NSK in both doorbell modes, device and
pinned-host buffers, ring wrap-around, idle exit + transparent relaunch,
stream ordering, stop with outstanding tickets."""
import time

import numpy as np
import pytest

import synth
from gpu_util import first_mismatch, kg_ready, oracle_pages, put

pytestmark = pytest.mark.gpu


@pytest.fixture
def nsk():
    kg, torch = kg_ready()
    yield kg, torch
    kg.nsk_stop()


def run(kg, torch, direction, mode, key, data, n, pb, ivs, where, inplace=False, stream=None, key_id=0):
    kg.set_key(key_id, key)
    tin = put(torch, data, where)
    tout = tin if inplace else (torch.empty_like(tin) if where == "device" else torch.empty_like(tin).pin_memory())
    tiv = None if ivs is None else put(torch, ivs, where)
    kg.wait(kg.submit_pages(direction, mode, tin, tout, n, pb, tiv, key_id, stream))
    (stream or torch.cuda.current_stream()).synchronize()
    return tout.cpu().numpy()


@pytest.mark.parametrize("flags", [0, 1])
@pytest.mark.parametrize("where", ["device", "pinned"])
def test_nsk_parity(nsk, flags, where):
    kg, torch = nsk
    kg.nsk_start(8, flags | kg.NSK_NOCAL, 5000)
    for (n, pb, kb) in [(1, 4096, 16), (16, 4096, 32), (33, 512, 24), (300, 4096, 16), (5, 16, 32), (1000, 48, 16)]:
        key = synth.make_key(kb, seed=n + pb)
        data = synth.make_pages(n, pb, seed=n * 7 + pb)
        ivs = synth.make_ivs(n, seed=n * 11)
        for d in (0, 1):
            for mode in (0, 1):
                exp = oracle_pages(d, mode, key, data, n, pb, ivs if mode == 0 else None)
                got = run(kg, torch, d, mode, key, data, n, pb, ivs if mode == 0 else None, where)
                assert first_mismatch(got, exp) is None, (n, pb, kb, d, mode)
        got = run(kg, torch, 1, 0, key, oracle_pages(0, 0, key, data, n, pb, ivs), n, pb, ivs, where, inplace=True)
        assert np.array_equal(got, data)


def test_nsk_ring_wraparound_and_many_inflight(nsk):
    kg, torch = nsk
    kg.nsk_start(4, kg.NSK_DIRECT | kg.NSK_NOCAL, 5000)
    n, pb = 4, 4096
    key = synth.make_key(16, seed=1)
    kg.set_key(0, key)
    data = synth.make_pages(n, pb, seed=2)
    ivs = synth.make_ivs(n, seed=3)
    exp = oracle_pages(0, 0, key, data, n, pb, ivs)
    src = torch.from_numpy(data).cuda()
    iv = torch.from_numpy(ivs).cuda()
    outs = [torch.empty_like(src) for _ in range(300)]
    tickets = [kg.submit_pages(0, 0, src, o, n, pb, iv, 0) for o in outs]   # > 64 ring slots
    assert all(b > a for a, b in zip(tickets, tickets[1:]))
    for t in tickets:
        kg.wait(t)
    for o in outs[::37] + [outs[-1]]:
        assert np.array_equal(o.cpu().numpy(), exp)


def test_nsk_idle_exit_and_relaunch(nsk):
    kg, torch = nsk
    kg.nsk_start(2, kg.NSK_DIRECT | kg.NSK_NOCAL, 30)        # 30 ms idle watchdog
    key = synth.make_key(16, seed=9)
    data = synth.make_pages(8, 4096, seed=10)
    ivs = synth.make_ivs(8, seed=11)
    exp = oracle_pages(1, 0, key, data, 8, 4096, ivs)
    l0 = kg.launch_count()
    for _ in range(3):
        assert np.array_equal(run(kg, torch, 1, 0, key, data, 8, 4096, ivs, "device"), exp)
        time.sleep(0.2)                        # the NSK exits; the next submit relaunches it
    assert kg.launch_count() - l0 >= 2


_IDLE_RACE = r"""
import random, sys, time
sys.path.insert(0, sys.argv[1])
import torch
import paper_1305_3345_b200 as kg
import synth
flags = int(sys.argv[2])
torch.cuda.set_device(0)
kg.init(0)
kg.set_key(0, synth.make_key(16, seed=5))
x = torch.from_numpy(synth.make_pages(1, 4096, seed=6)).cuda()
iv = torch.from_numpy(synth.make_ivs(1, seed=7)).cuda()
y = torch.empty_like(x)
ref = torch.empty_like(x)
kg.wait(kg.submit_pages(1, 0, x, ref, 1, 4096, iv, 0))
torch.cuda.synchronize()
kg.nsk_start(2, flags | kg.NSK_NOCAL, 1)                 # 1 ms idle watchdog
rnd = random.Random(11)
l0 = kg.launch_count()
for i in range(600):
    time.sleep(rnd.uniform(0.0006, 0.0016))  # straddle the watchdog
    kg.wait(kg.submit_pages(1, 0, x, y, 1, 4096, iv, 0))
torch.cuda.current_stream().synchronize()
assert torch.equal(y, ref)
print("relaunches", kg.launch_count() - l0)
kg.nsk_stop()
"""


@pytest.mark.parametrize("flags", [0, 1])
def test_nsk_idle_exit_race(tmp_path, flags):
    """a request posted while the NSK decides to exit on idle must
    not be lost.  Requests arrive at random gaps around a 1 ms watchdog; every
    one must complete (run in a subprocess with a timeout: a lost request
    would spin forever)."""
    import os
    import subprocess
    import sys
    kg_ready()
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "race.py"
    script.write_text(_IDLE_RACE)
    r = subprocess.run([sys.executable, str(script), root, str(flags)], capture_output=True, text=True, timeout=240)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert int(r.stdout.split("relaunches")[1]) >= 10   # the watchdog really fired between requests


def test_nsk_stream_ordering(nsk):
    """Ordered mode: the doorbell is rung by the stream after earlier work,
    and later work on the stream sees the result."""
    kg, torch = nsk
    kg.nsk_start(8, kg.NSK_NOCAL, 5000)
    n, pb = 2048, 4096
    key = synth.make_key(16, seed=20)
    kg.set_key(0, key)
    p = torch.from_numpy(synth.make_pages(n, pb, seed=21)).cuda()
    iv = torch.from_numpy(synth.make_ivs(n, seed=22)).cuda()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        a = torch.zeros_like(p)
        big = torch.ones(1 << 26, device="cuda")
        for _ in range(10):
            big.mul_(1.0001)
        a.copy_(p)
        c = torch.empty_like(a)
        kg.submit_pages(0, 0, a, c, n, pb, iv, 0, stream=s)
        back = torch.empty_like(a)
        t = kg.submit_pages(1, 0, c, back, n, pb, iv, 0, stream=s)
        ok = torch.equal(back, p)
    kg.wait(t)
    s.synchronize()
    assert bool(ok)


def test_nsk_stop_with_outstanding_and_restart(nsk):
    kg, torch = nsk
    kg.nsk_start(4, kg.NSK_DIRECT | kg.NSK_NOCAL, 5000)
    n, pb = 64, 4096
    kg.set_key(0, synth.make_key(16, seed=30))
    x = torch.from_numpy(synth.make_pages(n, pb, seed=31)).cuda()
    iv = torch.from_numpy(synth.make_ivs(n, seed=32)).cuda()
    y = torch.empty_like(x)
    ts = [kg.submit_pages(0, 0, x, y, n, pb, iv, 0) for _ in range(10)]
    kg.nsk_stop()
    for t in ts:
        kg.wait(t)                 # completed before the quit message
    lib = kg.raw_lib()
    assert lib.kg_nsk_stop() == kg.OK          # idempotent
    assert lib.kg_nsk_start(10 ** 6, 0, 0) == kg.EINVAL
    assert lib.kg_nsk_start(2, 8, 0) == kg.EINVAL
    kg.nsk_start(2, kg.NSK_NOCAL, 0)
    assert lib.kg_nsk_start(2, 0, 0) == kg.EINVAL   # already running
    ref = torch.empty_like(x)
    kg.wait(kg.submit_pages(0, 0, x, ref, n, pb, iv, 0))
    kg.nsk_stop()
    regular = torch.empty_like(x)
    kg.wait(kg.submit_pages(0, 0, x, regular, n, pb, iv, 0))   # launch-per-batch path again
    assert torch.equal(ref, regular) and torch.equal(y, regular)


def test_nsk_size_dispatch(nsk):
    """Row f2: small requests to the NSK, large ones launched on the free SMs."""
    kg, torch = nsk
    kg.nsk_start(16, kg.NSK_DIRECT, 5000)
    thr = kg.nsk_dispatch(0)                 # calibrate
    assert thr % 4096 == 0
    kg.nsk_dispatch(64 << 10)                # force: <= 16 pages to the NSK
    key = synth.make_key(16, seed=40)
    for n in (4, 16, 17, 3000):
        data = synth.make_pages(n, 4096, seed=n)
        ivs = synth.make_ivs(n, seed=n + 1)
        exp = oracle_pages(1, 0, key, data, n, 4096, ivs)
        l0 = kg.launch_count()
        got = run(kg, torch, 1, 0, key, data, n, 4096, ivs, "device")
        launched = kg.launch_count() - l0
        assert first_mismatch(got, exp) is None, n
        assert launched == (0 if n <= 16 else 1), (n, launched)
    # pinned + large goes through the staged path on the remaining SMs
    n = 5000
    data = synth.make_pages(n, 4096, seed=77)
    ivs = synth.make_ivs(n, seed=78)
    exp = oracle_pages(0, 0, key, data, n, 4096, ivs)
    assert first_mismatch(run(kg, torch, 0, 0, key, data, n, 4096, ivs, "pinned"), exp) is None


def test_nsk_multithreaded_soak(nsk):
    """Several host threads post to the NSK concurrently (ring wrap-around,
    completion words, waiter accounting); every ticket completes once and the
    outputs are right."""
    import threading
    kg, torch = nsk
    kg.nsk_start(8, kg.NSK_DIRECT | kg.NSK_NOCAL, 5000)
    n, pb = 16, 4096
    key = synth.make_key(16, seed=77)
    kg.set_key(3, key)
    data = synth.make_pages(n, pb, seed=78)
    ivs = synth.make_ivs(n, seed=79)
    exp = oracle_pages(1, 0, key, data, n, pb, ivs)
    src = torch.from_numpy(data).cuda()
    iv = torch.from_numpy(ivs).cuda()
    torch.cuda.current_stream().synchronize()
    errors, seen = [], []
    lock = threading.Lock()

    def worker(tid):
        try:
            outs = [torch.empty_like(src) for _ in range(3)]
            torch.cuda.current_stream().synchronize()
            for i in range(300):
                o = outs[i % 3]
                t = kg.submit_pages(1, 0, src, o, n, pb, iv, 3)
                with lock:
                    seen.append(t)
                kg.wait(t)
                if i % 71 == 0 and not np.array_equal(o.cpu().numpy(), exp):
                    errors.append((tid, i))
        except Exception as e:  # noqa: BLE001
            errors.append(repr(e))

    ths = [threading.Thread(target=worker, args=(k,)) for k in range(4)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    assert not errors, errors[:5]
    assert len(seen) == len(set(seen)) == 1200


@pytest.mark.parametrize("where", ["device", "pinned"])
def test_keyed_batches_while_nsk_runs(nsk, where):
    """Mixed-key batches are launched on the SMs the NSK leaves free (a grid
    over all SMs would wait behind the resident NSK forever)."""
    kg, torch = nsk
    kg.nsk_start(16, kg.NSK_DIRECT | kg.NSK_NOCAL, 5000)
    keys = {kid: synth.make_key(16, seed=300 + kid) for kid in (5, 6, 7)}
    for kid, k in keys.items():
        kg.set_key(kid, k)
    s = torch.cuda.Stream()
    for d, mode, n in ((1, 0, 3000), (0, 0, 700), (0, 1, 9000)):
        rng = np.random.default_rng(n)
        ids = np.array(list(keys), dtype=np.uint16)[rng.integers(0, 3, n)]
        data = synth.make_pages(n, 4096, seed=n + 3)
        ivs = synth.make_ivs(n, seed=n + 4) if mode == 0 else None
        exp = np.empty_like(data)
        for p in range(n):
            sl = slice(p * 4096, (p + 1) * 4096)
            exp[sl] = oracle_pages(d, mode, keys[int(ids[p])], data[sl], 1, 4096,
                                   None if ivs is None else ivs[16 * p:16 * p + 16])
        tin = put(torch, data, where)
        tout = torch.empty_like(tin) if where == "device" else torch.empty_like(tin).pin_memory()
        tiv = None if ivs is None else put(torch, ivs, where)
        tid = torch.from_numpy(ids.astype(np.int16)).cuda()
        s.synchronize()
        kg.wait(kg.submit_pages_keyed(d, mode, tin, tout, n, 4096, tiv, tid, 16, s))
        s.synchronize()
        assert first_mismatch(tout.cpu().numpy(), exp) is None, (d, mode, n)


def test_nsk_start_calibrates_and_dispatch_is_monotone(nsk):
    """Row f2 as built: kg_nsk_start calibrates the NSK/launch crossover at
    start (the paper's "calibrate it using microbenchmarks at boot time",
    PAPER.md:493-495); the threshold is kg_dispatch_threshold of the recorded
    samples, and the dispatch it implies is monotone: every request up to it
    goes to the NSK (no launch), every larger one is launched."""
    kg, torch = nsk
    kg.nsk_start(16, kg.NSK_DIRECT, 5000)
    pts = kg.nsk_calibration()
    assert len(pts) >= 2 and [p[0] for p in pts] == [4096 << i for i in range(len(pts))]
    assert all(p[1] > 0 and p[2] > 0 for p in pts)
    chosen = kg.dispatch_threshold(pts)
    key = synth.make_key(16, seed=60)
    kg.set_key(0, key)
    nmax = 1 << 13
    x = torch.from_numpy(synth.make_pages(nmax, 4096, seed=61)).cuda()
    iv = torch.from_numpy(synth.make_ivs(nmax, seed=62)).cuda()
    y = torch.empty_like(x)
    s = torch.cuda.current_stream()
    s.synchronize()
    routed = []
    for k in range(14):
        n = 1 << k
        l0 = kg.launch_count()
        kg.wait(kg.submit_pages(1, 0, x, y, n, 4096, iv, 0))
        routed.append(kg.launch_count() - l0 == 0)          # True: served by the NSK
        assert routed[-1] == (n * 4096 <= chosen), (n, chosen, pts)
    assert routed == sorted(routed, reverse=True)           # monotone
    s.synchronize()
    exp = oracle_pages(1, 0, key, x.cpu().numpy(), nmax, 4096, iv.cpu().numpy())
    assert first_mismatch(y.cpu().numpy(), exp) is None
