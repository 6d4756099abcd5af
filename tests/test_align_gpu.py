"""Buffers that are 16-byte aligned but not 32-byte aligned (kg.h promises
16).  The block-pair and wide chain kernels move two blocks with 256-bit
accesses that need 32-byte alignment (kg_internal.h wide_ok), so such
batches must take the one-block-per-lane kernels and still match the oracle
byte for byte -- for every kernel family, every memory kind and in place.
Also the constant-bank key race of mixed-key batches (a refill queued on a
busy stream, then a launch on an idle stream that must wait for it)."""
import numpy as np
import pytest

import synth
from gpu_util import first_mismatch, kg_ready, oracle_pages

pytestmark = pytest.mark.gpu


def offset_view(torch, nbytes, where, off):
    """A uint8 view of nbytes starting `off` bytes into a fresh allocation
    (torch allocations are >= 512-byte aligned, so off = 16 gives 16 mod 32)."""
    if where == "device":
        base = torch.empty(nbytes + 128, dtype=torch.uint8, device="cuda")
    else:
        base = torch.empty(nbytes + 128, dtype=torch.uint8).pin_memory()
    v = base[off:off + nbytes]
    assert v.data_ptr() % 32 == off % 32
    return v


CASES = [(1, 0), (0, 0), (1, 1), (0, 1)]  # (dir, mode): CBC dec, CBC enc, ECB dec, ECB enc


@pytest.mark.parametrize("direction,mode", CASES)
@pytest.mark.parametrize("in_off,out_off", [(16, 0), (0, 16), (16, 16), (48, 80)])
@pytest.mark.parametrize("key_bytes", [16, 32])
def test_misaligned_device(direction, mode, in_off, out_off, key_bytes):
    kg, torch = kg_ready()
    n, pb = 300, 4096
    key = synth.make_key(key_bytes, seed=401)
    kg.set_key(3, key)
    data = synth.make_pages(n, pb, seed=402)
    ivs = synth.make_ivs(n, seed=403) if mode == 0 else None
    exp = oracle_pages(direction, mode, key, data, n, pb, ivs)
    x = offset_view(torch, n * pb, "device", in_off)
    x.copy_(torch.from_numpy(data))
    out = offset_view(torch, n * pb, "device", out_off)
    iv = None if ivs is None else torch.from_numpy(ivs).cuda()
    kg.wait(kg.submit_pages(direction, mode, x, out, n, pb, iv, 3))
    torch.cuda.synchronize()
    assert first_mismatch(out.cpu().numpy(), exp) is None


@pytest.mark.parametrize("direction,mode", CASES)
def test_misaligned_in_place(direction, mode):
    kg, torch = kg_ready()
    n, pb = 150, 4096
    key = synth.make_key(16, seed=404)
    kg.set_key(3, key)
    data = synth.make_pages(n, pb, seed=405)
    ivs = synth.make_ivs(n, seed=406) if mode == 0 else None
    exp = oracle_pages(direction, mode, key, data, n, pb, ivs)
    x = offset_view(torch, n * pb, "device", 16)
    x.copy_(torch.from_numpy(data))
    iv = None if ivs is None else torch.from_numpy(ivs).cuda()
    kg.wait(kg.submit_pages(direction, mode, x, x, n, pb, iv, 3))
    torch.cuda.synchronize()
    assert first_mismatch(x.cpu().numpy(), exp) is None


@pytest.mark.parametrize("host_path", [0, 1])   # staged, zero-copy
@pytest.mark.parametrize("direction,mode", CASES)
def test_misaligned_pinned(host_path, direction, mode):
    kg, torch = kg_ready()
    n, pb = 64, 4096
    key = synth.make_key(16, seed=407)
    kg.set_key(3, key)
    data = synth.make_pages(n, pb, seed=408)
    ivs = synth.make_ivs(n, seed=409) if mode == 0 else None
    exp = oracle_pages(direction, mode, key, data, n, pb, ivs)
    x = offset_view(torch, n * pb, "pinned", 16)
    x.copy_(torch.from_numpy(data))
    out = offset_view(torch, n * pb, "pinned", 16)
    iv = None if ivs is None else torch.from_numpy(ivs).pin_memory()
    kg.set_host_path(host_path, 1 << 30)
    try:
        kg.wait(kg.submit_pages(direction, mode, x, out, n, pb, iv, 3))
    finally:
        kg.set_host_path(kg.HOST_AUTO, 32 << 20)
    torch.cuda.synchronize()
    assert first_mismatch(out.numpy(), exp) is None


@pytest.mark.parametrize("direction,mode", CASES)
@pytest.mark.parametrize("where", ["device", "pinned"])
def test_misaligned_keyed(direction, mode, where):
    kg, torch = kg_ready()
    n, pb = 200, 4096
    keys = {i: synth.make_key(16, seed=410 + i) for i in (30, 31, 32)}
    for k, v in keys.items():
        kg.set_key(k, v)
    rng = np.random.default_rng(411)
    ids = np.array(list(keys), dtype=np.uint16)[rng.integers(0, 3, n)]
    data = synth.make_pages(n, pb, seed=412)
    ivs = synth.make_ivs(n, seed=413) if mode == 0 else None
    exp = np.empty_like(data)
    for p in range(n):
        sl = slice(p * pb, (p + 1) * pb)
        exp[sl] = oracle_pages(direction, mode, keys[int(ids[p])], data[sl], 1, pb,
                               None if ivs is None else ivs[16 * p:16 * p + 16])
    x = offset_view(torch, n * pb, where, 16)
    x.copy_(torch.from_numpy(data))
    out = offset_view(torch, n * pb, where, 16)
    dev = "cuda" if where == "device" else "cpu"
    tid = torch.from_numpy(ids.astype(np.int16)).to(dev)
    iv = None if ivs is None else torch.from_numpy(ivs).to(dev)
    if where == "pinned":
        tid = tid.pin_memory()
        iv = None if iv is None else iv.pin_memory()
    kg.wait(kg.submit_pages_keyed(direction, mode, x, out, n, pb, iv, tid, 16))
    torch.cuda.synchronize()
    assert first_mismatch(out.cpu().numpy(), exp) is None


def test_const_key_refill_on_busy_stream_then_idle_stream():
    """the constant-bank key copy is refilled on stream A behind a
    long kernel; a launch on idle stream B with the same snapshot must wait
    for that refill instead of reading the previous keys."""
    kg, torch = kg_ready()
    n, pb = 512, 4096
    k_old, k_new = synth.make_key(16, seed=420), synth.make_key(16, seed=421)
    kg.set_key(40, k_old)
    data = synth.make_pages(n, pb, seed=422)
    ivs = synth.make_ivs(n, seed=423)
    x = torch.from_numpy(data).cuda()
    iv = torch.from_numpy(ivs).cuda()
    ids = torch.full((n,), 40, dtype=torch.int16, device="cuda")
    out0 = torch.empty_like(x)
    kg.wait(kg.submit_pages_keyed(1, 0, x, out0, n, pb, iv, ids, 16))   # constant bank: k_old (decrypt)
    torch.cuda.synchronize()
    kg.set_key(40, k_new)                                                 # new snapshot version
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    out_a, out_b = torch.empty_like(x), torch.empty_like(x)
    with torch.cuda.stream(sa):
        torch.cuda._sleep(50_000_000)                                     # ~25 ms busy on A
    ta = kg.submit_pages_keyed(1, 0, x, out_a, n, pb, iv, ids, 16, sa)     # refill queued behind the sleep
    tb = kg.submit_pages_keyed(1, 0, x, out_b, n, pb, iv, ids, 16, sb)     # same snapshot, idle stream
    kg.wait(tb)
    kg.wait(ta)
    torch.cuda.synchronize()
    exp = oracle_pages(1, 0, k_new, data, n, pb, ivs)
    assert first_mismatch(out_a.cpu().numpy(), exp) is None
    assert first_mismatch(out_b.cpu().numpy(), exp) is None
