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
        kg.set_pipeline(0, 4)
        kg.set_host_path(kg.HOST_AUTO, 32 << 20)
    from gpu_util import oracle_pages
    assert np.array_equal(hout.numpy(), oracle_pages(1, 0, key, data, n, pb, ivs))


_FAULT = r"""
import os, sys
sys.path.insert(0, sys.argv[1])
import numpy as np
import torch
import paper_1305_3345_b200 as kg
import oracle, synth
torch.cuda.set_device(0)
kg.init(0)
kg.set_key(0, synth.make_key(16))
small = torch.zeros(1 << 20, dtype=torch.uint8, device="cuda")
torch.cuda.synchronize()
# an ECB batch that runs 3 GiB past a 1 MiB allocation (48-byte pages: plain loads)
t = kg.submit_pages(1, 1, small, small, 1 << 26, 48, None, 0)
assert t >= 0
rc = kg.wait_raw(t)
print("wait", rc)
assert rc == kg.ECUDA
assert kg.submit_pages_raw(1, 1, small, small, 1, 48, None, 0) in (kg.ECUDA, kg.EINVAL)
lib = kg.raw_lib()
assert lib.kg_shutdown() == kg.OK          # resets the faulted context
assert lib.kg_init(0) == kg.OK             # ... and the library starts over
key = synth.make_key(16, seed=3)
kg.set_key(0, key)
n, pb = 8, 4096
data, ivs = synth.make_pages(n, pb, seed=4), synth.make_ivs(n, seed=5)
hx, hout, hiv = kg.alloc_pinned(n * pb), kg.alloc_pinned(n * pb), kg.alloc_pinned(16 * n)
hx.copy_(torch.from_numpy(data)); hiv.copy_(torch.from_numpy(ivs))
kg.wait(kg.submit_pages(1, 0, hx, hout, n, pb, hiv, 0))     # pinned host: zero-copy launch in the new context
assert np.array_equal(hout.numpy(), oracle.pages(1, 0, key, data, n, pb, ivs))
print("recovered")
sys.stdout.flush()
os._exit(0)
"""


def test_ecuda_async_fault_then_shutdown_init_recovers(tmp_path):
    """An asynchronous device fault surfaces as KG_ECUDA at kg_wait;
    kg_shutdown + kg_init recover (in a subprocess: the fault kills that
    process's context)."""
    import os
    import subprocess
    import sys
    kg_ready()
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    f = tmp_path / "fault.py"
    f.write_text(_FAULT)
    r = subprocess.run([sys.executable, str(f), root], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "recovered" in r.stdout, r.stdout[-2000:] + r.stderr[-3000:]
