"""Every KG_E* condition of include/kg.h is detected synchronously and
writes nothing; tickets are strictly increasing; double wait -> KG_ETICKET."""
import ctypes

import numpy as np
import pytest

import synth
from gpu_util import kg_ready

pytestmark = pytest.mark.gpu


@pytest.fixture
def env():
    kg, torch = kg_ready()
    kg.set_key(0, synth.make_key(16))
    n, pb = 8, 4096
    buf = torch.zeros(3 * n * pb + 64, dtype=torch.uint8, device="cuda")
    x = buf[:n * pb]
    out = buf[n * pb:2 * n * pb]
    iv = torch.zeros(16 * n, dtype=torch.uint8, device="cuda")
    return kg, torch, buf, x, out, iv, n, pb


def rc(kg, *a):
    return kg.submit_pages_raw(*a)


def test_einval_cases(env):
    kg, torch, buf, x, out, iv, n, pb = env
    E = kg.EINVAL
    sentinel = out.clone()
    assert rc(kg, 2, 0, x, out, n, pb, iv, 0) == E                 # bad dir
    assert rc(kg, -1, 0, x, out, n, pb, iv, 0) == E
    assert rc(kg, 0, 2, x, out, n, pb, iv, 0) == E                 # bad mode
    assert rc(kg, 0, 0, x, out, 0, pb, iv, 0) == E                 # empty batch
    assert rc(kg, 0, 0, x, out, n, 0, iv, 0) == E                  # page_bytes 0
    assert rc(kg, 0, 0, x, out, n, 4095, iv, 0) == E               # not a multiple of 16
    assert rc(kg, 0, 0, x, out, 1 << 60, 4096, iv, 0) == E         # overflow 64 bits
    assert rc(kg, 0, 0, None, out, n, pb, iv, 0) == E              # NULL
    assert rc(kg, 0, 0, x, None, n, pb, iv, 0) == E
    assert rc(kg, 0, 0, x, out, n, pb, None, 0) == E               # CBC needs IVs
    assert rc(kg, 0, 0, x.data_ptr() + 8, out, n, pb, iv, 0) == E  # misaligned
    assert rc(kg, 0, 0, x, out.data_ptr() + 4, n, pb, iv, 0) == E
    assert rc(kg, 0, 0, x, out, n, pb, iv.data_ptr() + 1, 0) == E
    assert rc(kg, 0, 0, x, x.data_ptr() + 4096, n, pb, iv, 0) == E  # partial overlap
    assert rc(kg, 0, 0, x.data_ptr() + 4096, x, n, pb, iv, 0) == E
    assert rc(kg, 0, 0, x, out, n, pb, out.data_ptr() + 32, 0) == E  # ivs inside out
    assert rc(kg, 0, 0, x, out, n, pb, iv, -1) == E                # key id range
    assert rc(kg, 0, 0, x, out, n, pb, iv, kg.MAX_KEYS) == E
    pageable = np.zeros(n * pb + 16, dtype=np.uint8)
    addr = (pageable.ctypes.data + 15) & ~15
    assert rc(kg, 0, 0, addr, out, n, pb, iv, 0) == E              # pageable host memory
    assert rc(kg, 0, 0, x, addr, n, pb, iv, 0) == E
    torch.cuda.synchronize()
    assert torch.equal(out, sentinel)                              # nothing written


def test_ecb_accepts_null_ivs(env):
    kg, torch, buf, x, out, iv, n, pb = env
    t = rc(kg, 0, 1, x, out, n, pb, None, 0)
    assert t >= 0
    kg.wait(t)


def test_enokey_and_key_errors(env):
    kg, torch, buf, x, out, iv, n, pb = env
    # a fresh key table (other test files may have set id 200 in this process)
    torch.cuda.synchronize()
    assert kg.raw_lib().kg_shutdown() == kg.OK
    kg.init(0)
    kg.set_key(0, synth.make_key(16))
    assert rc(kg, 0, 0, x, out, n, pb, iv, 200) == kg.ENOKEY
    lib = kg.raw_lib()
    assert lib.kg_set_key(0, b"\0" * 20, 20) == kg.EINVAL
    assert lib.kg_set_key(0, None, 16) == kg.EINVAL
    assert lib.kg_set_key(kg.MAX_KEYS, b"\0" * 16, 16) == kg.EINVAL
    assert lib.kg_set_key(-1, b"\0" * 16, 16) == kg.EINVAL
    for kb in (16, 24, 32):
        assert lib.kg_set_key(1, b"\1" * kb, kb) == kg.OK


def test_tickets_monotonic_and_retire(env):
    kg, torch, buf, x, out, iv, n, pb = env
    ts = [kg.submit_pages(0, 0, x, out, n, pb, iv, 0) for _ in range(50)]
    assert all(b > a for a, b in zip(ts, ts[1:]))
    for t in ts:
        kg.wait(t)
    assert kg.wait_raw(ts[0]) == kg.ETICKET
    assert kg.poll_raw(ts[-1]) == kg.ETICKET
    assert kg.wait_raw(10 ** 15) == kg.ETICKET
    assert kg.wait_raw(-5) == kg.ETICKET


def test_init_other_device_rejected(env):
    kg, torch, *_ = env
    lib = kg.raw_lib()
    assert lib.kg_init(0) == kg.OK          # idempotent
    assert lib.kg_init(1 if torch.cuda.device_count() > 1 else 999) == kg.EINVAL
    assert lib.kg_set_pipeline(8, 3) == kg.EINVAL          # 0 = auto is valid; 1..15 are not
    assert lib.kg_set_pipeline(1 << 20, 1) == kg.EINVAL
    assert lib.kg_set_pipeline(1 << 20, 9) == kg.EINVAL


def test_shutdown_and_reinit():
    kg, torch = kg_ready()
    kg.set_key(3, synth.make_key(16))
    kg.shutdown()
    lib = kg.raw_lib()
    assert lib.kg_shutdown() == kg.ENOTINIT
    kg.init(0)
    x = torch.zeros(4096, dtype=torch.uint8, device="cuda")
    iv = torch.zeros(16, dtype=torch.uint8, device="cuda")
    assert kg.submit_pages_raw(0, 0, x, x, 1, 4096, iv, 3) == kg.ENOKEY   # keys forgotten


def test_eagain_ticket_table_full():
    """KG_MAX_INFLIGHT unretired tickets: the next submit returns KG_EAGAIN
    (SPEC.md:51 QueueFull) and enqueues nothing; waiting on the oldest frees
    a slot."""
    kg, torch = kg_ready()
    kg.set_key(0, synth.make_key(16))
    x = torch.zeros(16, dtype=torch.uint8, device="cuda")
    y = torch.zeros(16, dtype=torch.uint8, device="cuda")
    l0 = kg.launch_count()
    ts = [kg.submit_pages(1, 1, x, y, 1, 16, None, 0) for _ in range(kg.MAX_INFLIGHT)]
    launched = kg.launch_count() - l0
    assert kg.submit_pages_raw(1, 1, x, y, 1, 16, None, 0) == kg.EAGAIN
    assert kg.launch_count() - l0 == launched                  # nothing enqueued
    kg.wait(ts[0])
    t = kg.submit_pages(1, 1, x, y, 1, 16, None, 0)
    assert t > ts[-1]
    for tk in ts[1:] + [t]:
        kg.wait(tk)


def test_enomem_staging_then_recovers():
    """The device staging ring cannot be allocated -> KG_ENOMEM, nothing
    written; once memory is free again the same batch succeeds."""
    kg, torch = kg_ready()
    key = synth.make_key(16)
    kg.set_key(0, key)
    n, pb = 4096, 4096
    data = synth.make_pages(n, pb, seed=90)
    ivs = synth.make_ivs(n, seed=91)
    hx = torch.from_numpy(data).pin_memory()
    hiv = torch.from_numpy(ivs).pin_memory()
    hout = torch.zeros(n * pb, dtype=torch.uint8).pin_memory()
    kg.set_host_path(kg.HOST_STAGED, 0)
    kg.set_pipeline(n * pb, 3)                     # slot count changes: the ring is freed and re-allocated on use
    torch.cuda.empty_cache()
    free, _ = torch.cuda.mem_get_info()
    hog = torch.empty(free - (24 << 20), dtype=torch.uint8, device="cuda")   # leave < 3 x 16 MiB
    try:
        assert kg.submit_pages_raw(1, 0, hx, hout, n, pb, hiv, 0) == kg.ENOMEM
        assert int(hout.sum()) == 0                # nothing written
    finally:
        del hog
        torch.cuda.empty_cache()
    try:
        kg.wait(kg.submit_pages(1, 0, hx, hout, n, pb, hiv, 0))
    finally:
        kg.set_pipeline(0, kg.DEFAULT_STAGING_SLOTS)
        kg.set_host_path(kg.HOST_AUTO, 32 << 20)
    from gpu_util import oracle_pages
    assert np.array_equal(hout.numpy(), oracle_pages(1, 0, key, data, n, pb, ivs))


_FAULT = r"""
import os, sys
sys.path.insert(0, sys.argv[1])
import torch                    # CPU tensors only: the library owns this process's CUDA context
import paper_1305_3345_b200 as kg
import synth
lib = kg.raw_lib()
assert lib.kg_init(0) == kg.OK
kg.set_key(0, synth.make_key(16))
kg.set_host_path(kg.HOST_ZEROCOPY, 0)
small = kg.alloc_pinned(1 << 20)
ok_in, ok_out = kg.alloc_pinned(4096), kg.alloc_pinned(4096)
# an ECB batch that runs 3 GiB past a 1 MiB pinned allocation, read and
# written in place over its device mapping (48-byte pages: plain loads),
# followed by a well-formed batch
bad = kg.submit_pages(1, 1, small, small, 1 << 26, 48, None, 0)
good = kg.submit_pages(1, 1, ok_in, ok_out, 1, 4096, None, 0)
print("wait_bad", kg.wait_raw(bad))
print("poll_good", kg.poll_raw(good))
print("wait_good", kg.wait_raw(good))
print("submit_after", kg.submit_pages_raw(1, 1, ok_in, ok_out, 1, 4096, None, 0))
print("shutdown", lib.kg_shutdown())
print("init_after", lib.kg_init(0))
sys.stdout.flush()
os._exit(0)
"""

_FRESH = r"""
import sys
sys.path.insert(0, sys.argv[1])
import numpy as np, torch
import paper_1305_3345_b200 as kg
import oracle, synth
kg.init(0)
key = synth.make_key(16, seed=3)
kg.set_key(0, key)
n, pb = 8, 4096
data, ivs = synth.make_pages(n, pb, seed=4), synth.make_ivs(n, seed=5)
x, iv = torch.from_numpy(data).cuda(), torch.from_numpy(ivs).cuda()
y = torch.empty_like(x)
kg.wait(kg.submit_pages(1, 0, x, y, n, pb, iv, 0))
assert np.array_equal(y.cpu().numpy(), oracle.pages(1, 0, key, data, n, pb, ivs))
print("fresh ok")
"""


def test_ecuda_async_fault_is_reported_and_terminal(tmp_path):
    """An asynchronous device fault surfaces as KG_ECUDA at kg_wait (and for
    every later ticket and submit of the process); kg_shutdown still succeeds;
    the dead context makes kg_init return KG_ECUDA (CUDA's sticky errors end
    only with the process); a new process then runs correctly (kg.h)."""
    import os
    import subprocess
    import sys
    kg, _ = kg_ready()
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    f = tmp_path / "fault.py"
    f.write_text(_FAULT)
    r = subprocess.run([sys.executable, str(f), root], capture_output=True, text=True, timeout=300)
    out = dict(l.split() for l in r.stdout.splitlines() if len(l.split()) == 2)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    assert int(out["wait_bad"]) == kg.ECUDA
    assert int(out["poll_good"]) == kg.ECUDA and int(out["wait_good"]) == kg.ECUDA
    assert int(out["submit_after"]) == kg.ECUDA
    assert int(out["shutdown"]) == kg.OK
    assert int(out["init_after"]) == kg.ECUDA
    g = tmp_path / "fresh.py"
    g.write_text(_FRESH)
    r = subprocess.run([sys.executable, str(g), root], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "fresh ok" in r.stdout, r.stdout[-2000:] + r.stderr[-3000:]
