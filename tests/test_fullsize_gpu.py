"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py
times, against the ORACLE on every byte:
  C2  AES-128-CBC decrypt, 65,536 x 4 KiB (256 MiB), device and pinned host;
  C3  AES-256-CBC encrypt, 262,144 x 4 KiB (1 GiB);
  C4  AES-128-CBC decrypt at 1 GiB (the top of the sweep; also the round trip of C3's size);
  C5  AES-128-CBC decrypt of 64 GiB in place: page p holds page p mod M of a
      seeded M = 65,537-page set; the oracle decrypts the
      M pages once and every byte of the 64 GiB is compared on the device
      against the oracle's page (p mod M).
The oracle runs on all host cores (its results do not depend on the thread
count: tests/test_oracle_invariants.py)."""
import numpy as np
import pytest

import synth
from gpu_util import first_mismatch, kg_ready, oracle_pages

pytestmark = pytest.mark.gpu
PB = 4096
_CACHE = {}


def oracle_full(name, direction, key, data, n, ivs):
    if name not in _CACHE:
        _CACHE[name] = oracle_pages(direction, 0, key, data, n, PB, ivs)
    return _CACHE[name]


def c2_inputs():
    n = 65536
    return n, synth.make_key(16), synth.make_pages(n, PB), synth.make_ivs(n)


@pytest.mark.parametrize("where", ["device", "pinned"])
def test_c2_decrypt_256mib_every_byte(where):
    kg, torch = kg_ready()
    n, key, data, ivs = c2_inputs()
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
    exp = oracle_full("c2", 1, key, data, n, ivs)
    assert first_mismatch(out.cpu().numpy(), exp) is None


def test_c3_encrypt_1gib_aes256_every_byte():
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
    exp = oracle_full("c3", 0, key, data, n, ivs)
    assert first_mismatch(out.cpu().numpy(), exp) is None
    # C4 at 1 GiB: AES-128 decrypt of the same 262,144 pages, every byte vs the oracle
    key16 = synth.make_key(16)
    kg.set_key(0, key16)
    kg.wait(kg.submit_pages(1, 0, x, out, n, PB, iv, 0))
    torch.cuda.synchronize()
    exp4 = oracle_pages(1, 0, key16, data, n, PB, ivs)
    assert first_mismatch(out.cpu().numpy(), exp4) is None


def test_c5_decrypt_64gib_in_place_every_byte():
    """16,777,216 pages (2^32 blocks) in place, 17 texture windows per launch.
    Expected page p = the oracle's decryption of pattern page p mod M."""
    kg, torch = kg_ready()
    free, _ = torch.cuda.mem_get_info()
    n, M = 16777216, 65537
    if free < n * PB + (4 << 30):
        pytest.skip("needs ~70 GB of free HBM")
    key = synth.make_key(16, seed=55)
    pat_np = synth.make_pages(M, PB, seed=56)
    ivp_np = synth.make_ivs(M, seed=57)
    exp_np = oracle_pages(1, 0, key, pat_np, M, PB, ivp_np)       # the oracle, not the GPU
    kg.set_key(2, key)
    pat = torch.from_numpy(pat_np).cuda().view(M, PB)
    ivp = torch.from_numpy(ivp_np).cuda().view(M, 16)
    big = torch.empty((n, PB), dtype=torch.uint8, device="cuda")
    ivs = torch.empty((n, 16), dtype=torch.uint8, device="cuda")
    for s in range(0, n, M):
        e = min(n, s + M)
        big[s:e].copy_(pat[:e - s])
        ivs[s:e].copy_(ivp[:e - s])
    del pat, ivp
    kg.wait(kg.submit_pages(1, 0, big, big, n, PB, ivs, 2))
    torch.cuda.synchronize()
    exp = torch.from_numpy(exp_np).cuda().view(M, PB)
    bad_pages = 0
    first_bad = None
    for s in range(0, n, M):
        e = min(n, s + M)
        neq = (big[s:e] != exp[:e - s]).any(dim=1)
        c = int(neq.sum())
        if c and first_bad is None:
            first_bad = s + int(torch.nonzero(neq)[0])
        bad_pages += c
    assert bad_pages == 0, f"{bad_pages} pages differ from the oracle, first {first_bad}"
    # the last page (block index 2^32 - 1) once more, through host memory
    p = n - 1
    assert np.array_equal(big[p].cpu().numpy(), exp_np[(p % M) * PB:(p % M + 1) * PB])
    del big, ivs, exp
    torch.cuda.empty_cache()
