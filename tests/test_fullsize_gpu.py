"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py
times, on sampled pages the oracle computes one by one (plus the pages at
every CTA-range boundary), and via page-locality properties that hold at any
size for the 64 GiB case."""
import numpy as np
import pytest

import synth
from gpu_util import kg_ready, oracle_pages

pytestmark = pytest.mark.gpu
PB = 4096


def sample_pages(n, k=96, seed=0, sms=148):
    rng = np.random.default_rng(seed)
    s = set(rng.integers(0, n, k).tolist())
    s |= {0, 1, n - 2, n - 1}
    for c in range(1, sms):            # CTA range boundaries (balanced split)
        b = (n * c) // sms
        s |= {b - 1, b}
    return sorted(p for p in s if 0 <= p < n)


def check_sampled(direction, key, data_np, ivs_np, out_np, pages):
    for p in pages:
        exp = oracle_pages(direction, 0, key, data_np[p * PB:(p + 1) * PB], 1, PB, ivs_np[16 * p:16 * p + 16])
        got = out_np[p * PB:(p + 1) * PB]
        assert np.array_equal(got, exp), f"page {p}"


@pytest.mark.parametrize("where", ["device", "pinned"])
def test_c2_decrypt_256mib(where):
    kg, torch = kg_ready()
    n = 65536
    key = synth.make_key(16)
    data = synth.make_pages(n, PB)
    ivs = synth.make_ivs(n)
    kg.set_key(0, key)
    if where == "device":
        x = torch.from_numpy(data).cuda()
        iv = torch.from_numpy(ivs).cuda()
        out = torch.empty_like(x)
    else:
        x = torch.from_numpy(data).pin_memory()
        iv = torch.from_numpy(ivs).pin_memory()
        out = torch.empty(n * PB, dtype=torch.uint8).pin_memory()
    kg.wait(kg.submit_pages(1, 0, x, out, n, PB, iv, 0))
    torch.cuda.synchronize()
    check_sampled(1, key, data, ivs, out.cpu().numpy(), sample_pages(n))


def test_c3_encrypt_1gib_aes256():
    kg, torch = kg_ready()
    n = 262144
    key = synth.make_key(32)
    data = synth.make_pages(n, PB)
    ivs = synth.make_ivs(n)
    kg.set_key(1, key)
    x = torch.from_numpy(data).cuda()
    iv = torch.from_numpy(ivs).cuda()
    out = torch.empty_like(x)
    kg.wait(kg.submit_pages(0, 0, x, out, n, PB, iv, 1))
    torch.cuda.synchronize()
    check_sampled(0, key, data, ivs, out.cpu().numpy(), sample_pages(n, seed=1))
    # round trip at full size on the device
    back = torch.empty_like(x)
    kg.wait(kg.submit_pages(1, 0, out, back, n, PB, iv, 1))
    assert torch.equal(back, x)


def test_c5_decrypt_64gib_in_place():
    """16,777,216 pages (2^32 blocks) in place.  Page p holds page p mod M of a
    seeded M = 65,537-page set (odd, so it never aliases power-of-two or CTA
    boundaries).  Every byte is compared on the device against the M-page
    run (pages are independent: a page's output depends only on its own bytes
    and IV), and that run is checked against the oracle on sampled pages."""
    kg, torch = kg_ready()
    free, _ = torch.cuda.mem_get_info()
    n, M = 16777216, 65537
    if free < n * PB + (4 << 30):
        pytest.skip("needs ~70 GB of free HBM")
    key = synth.make_key(16, seed=55)
    kg.set_key(2, key)
    pat = torch.from_numpy(synth.make_pages(M, PB, seed=56)).cuda().view(M, PB)
    ivp = torch.from_numpy(synth.make_ivs(M, seed=57)).cuda().view(M, 16)
    big = torch.empty((n, PB), dtype=torch.uint8, device="cuda")
    ivs = torch.empty((n, 16), dtype=torch.uint8, device="cuda")
    for s in range(0, n, M):
        e = min(n, s + M)
        big[s:e].copy_(pat[:e - s])
        ivs[s:e].copy_(ivp[:e - s])
    kg.wait(kg.submit_pages(1, 0, big, big, n, PB, ivs, 2))
    ref = torch.empty_like(pat)
    kg.wait(kg.submit_pages(1, 0, pat, ref, M, PB, ivp, 2))
    torch.cuda.synchronize()
    bad = 0
    for s in range(0, n, M):
        e = min(n, s + M)
        bad += int((big[s:e] != ref[:e - s]).any(dim=1).sum())
    assert bad == 0
    pat_np, ivp_np, ref_np = pat.cpu().numpy().reshape(-1), ivp.cpu().numpy().reshape(-1), ref.cpu().numpy().reshape(-1)
    check_sampled(1, key, pat_np, ivp_np, ref_np, sample_pages(M, k=48, seed=2))
    # spot-check big pages directly too (incl. the last page, block index 2^32-1)
    big_pages = [0, n // 2 + 3, n - 1]
    for p in big_pages:
        got = big[p].cpu().numpy()
        exp = oracle_pages(1, 0, key, pat_np[(p % M) * PB:(p % M + 1) * PB], 1, PB, ivp_np[16 * (p % M):16 * (p % M) + 16])
        assert np.array_equal(got, exp), p
    del big, ivs
    torch.cuda.empty_cache()
