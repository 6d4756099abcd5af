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
