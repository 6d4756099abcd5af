"""Properties of the CUDA path that hold at any size (SURVEY.md §8c
invariants), checked GPU-only (no oracle): round trip, decrypt locality incl.
the page boundary, encrypt propagation, page-permutation equivariance,
in-place == out-of-place, re-keying does not affect in-flight batches, and
stream ordering."""
import numpy as np
import pytest

import synth
from gpu_util import gpu_pages, kg_ready

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("key_bytes", [16, 24, 32])
def test_round_trip(key_bytes):
    n, pb = 3001, 4096
    key = synth.make_key(key_bytes, seed=key_bytes)
    p = synth.make_pages(n, pb, seed=1)
    iv = synth.make_ivs(n, seed=2)
    c = gpu_pages(0, 0, key, p, n, pb, iv)
    assert not np.array_equal(c, p)
    assert np.array_equal(gpu_pages(1, 0, key, c, n, pb, iv), p)
    e = gpu_pages(0, 1, key, p, n, pb, None)
    assert np.array_equal(gpu_pages(1, 1, key, e, n, pb, None), p)


def test_decrypt_locality_page_boundary():
    n, pb = 400, 4096
    m = pb // 16
    key = synth.make_key(16, seed=3)
    c = synth.make_pages(n, pb, seed=4)
    iv = synth.make_ivs(n, seed=5)
    p = gpu_pages(1, 0, key, c, n, pb, iv)
    for pg, j in [(0, 0), (150, 31), (150, 32), (299, m - 1), (n - 1, m - 1)]:
        c2 = c.copy()
        byte = pg * pb + 16 * j + 7
        c2[byte] ^= 0x04
        p2 = gpu_pages(1, 0, key, c2, n, pb, iv)
        blocks = set((np.nonzero(p != p2)[0] // 16).tolist())
        g = pg * m + j
        assert g in blocks
        if j + 1 < m:
            assert blocks == {g, g + 1}
            assert p2[byte + 16] ^ p[byte + 16] == 0x04
        else:
            assert blocks == {g}


def test_encrypt_propagation_stays_in_page():
    n, pb = 200, 4096
    m = pb // 16
    key = synth.make_key(32, seed=8)
    p = synth.make_pages(n, pb, seed=9)
    iv = synth.make_ivs(n, seed=10)
    c = gpu_pages(0, 0, key, p, n, pb, iv)
    pg, j = 123, 200
    p2 = p.copy()
    p2[pg * pb + 16 * j] ^= 1
    c2 = gpu_pages(0, 0, key, p2, n, pb, iv)
    blocks = sorted(set((np.nonzero(c != c2)[0] // 16).tolist()))
    assert blocks == list(range(pg * m + j, (pg + 1) * m))


def test_permutation_equivariance():
    n, pb = 500, 1024
    key = synth.make_key(16, seed=11)
    p = synth.make_pages(n, pb, seed=12)
    iv = synth.make_ivs(n, seed=13)
    perm = np.random.default_rng(0).permutation(n)
    for d in (0, 1):
        c = gpu_pages(d, 0, key, p, n, pb, iv)
        cp = gpu_pages(d, 0, key, p.reshape(n, pb)[perm].reshape(-1), n, pb, iv.reshape(n, 16)[perm].reshape(-1))
        assert np.array_equal(cp.reshape(n, pb), c.reshape(n, pb)[perm])


def test_rekey_does_not_affect_submitted_batch():
    kg, torch = kg_ready()
    n, pb = 2000, 4096
    k1, k2 = synth.make_key(16, seed=20), synth.make_key(16, seed=21)
    p = torch.from_numpy(synth.make_pages(n, pb, seed=22)).cuda()
    iv = torch.from_numpy(synth.make_ivs(n, seed=23)).cuda()
    o1 = torch.empty_like(p)
    o2 = torch.empty_like(p)
    kg.set_key(5, k1)
    t1 = kg.submit_pages(0, 0, p, o1, n, pb, iv, 5)
    kg.set_key(5, k2)            # re-key while t1 may still be running
    t2 = kg.submit_pages(0, 0, p, o2, n, pb, iv, 5)
    kg.wait(t1)
    kg.wait(t2)
    ref1 = gpu_pages(0, 0, k1, p.cpu().numpy(), n, pb, iv.cpu().numpy(), key_id=6)
    ref2 = gpu_pages(0, 0, k2, p.cpu().numpy(), n, pb, iv.cpu().numpy(), key_id=6)
    assert np.array_equal(o1.cpu().numpy(), ref1)
    assert np.array_equal(o2.cpu().numpy(), ref2)


def test_stream_ordering():
    """Work enqueued on the caller's stream before the submit is seen by the
    kernel; work after it sees the outputs (kg.h ordering contract)."""
    kg, torch = kg_ready()
    n, pb = 4096, 4096
    key = synth.make_key(16, seed=30)
    kg.set_key(0, key)
    p = synth.make_pages(n, pb, seed=31)
    iv = torch.from_numpy(synth.make_ivs(n, seed=32)).cuda()
    src = torch.from_numpy(p).cuda()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        a = torch.zeros(n * pb, dtype=torch.uint8, device="cuda")
        big = torch.ones(1 << 28, dtype=torch.float32, device="cuda")
        for _ in range(20):
            big.mul_(1.0001)          # keep the stream busy before the copy
        a.copy_(src)
        out = torch.empty_like(a)
        t = kg.submit_pages(0, 0, a, out, n, pb, iv, 0, stream=s)
        back = torch.empty_like(a)
        kg.submit_pages(1, 0, out, back, n, pb, iv, 0, stream=s)
        same = torch.equal(back, src)
    kg.wait(t)
    torch.cuda.synchronize()
    assert same


def test_poll_then_wait():
    kg, torch = kg_ready()
    n, pb = 1000, 4096
    kg.set_key(0, synth.make_key(16))
    x = torch.from_numpy(synth.make_pages(n, pb)).cuda()
    iv = torch.from_numpy(synth.make_ivs(n)).cuda()
    t = kg.submit_pages(1, 0, x, x, n, pb, iv, 0)
    while not kg.poll(t):
        pass
    kg.wait(t)
    assert kg.wait_raw(t) == kg.ETICKET
