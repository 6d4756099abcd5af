"""Randomised parity sweep: random (direction, mode, key size, page count,
page size, residency, in-place, host path) cases, each compared byte for byte
with the oracle.  Sizes stay small so the oracle finishes quickly."""
import os

import numpy as np
import pytest

import synth
from gpu_util import first_mismatch, gpu_pages, kg_ready, oracle_pages

pytestmark = pytest.mark.gpu


def test_random_cases():
    kg, torch = kg_ready()
    # KG_FUZZ_CASES / KG_FUZZ_SEED: longer soak runs (tools/runs/gpu_fuzz_soak.sh)
    rng = np.random.default_rng(int(os.environ.get("KG_FUZZ_SEED", "20261017")))
    for case in range(int(os.environ.get("KG_FUZZ_CASES", "150"))):
        d = int(rng.integers(0, 2))
        mode = int(rng.integers(0, 2))
        kb = int(rng.choice([16, 24, 32]))
        n = int(rng.choice([1, 2, 3, 5, 17, 31, 64, 149, 150, 300, 1000]))
        pb = 16 * int(rng.choice([1, 2, 3, 4, 7, 16, 31, 32, 33, 64, 128, 256, 512]))
        if n * pb > (4 << 20):
            n = max(1, (4 << 20) // pb)
        where = str(rng.choice(["device", "pinned"]))
        inplace = bool(rng.integers(0, 2))
        hp = int(rng.integers(0, 3))
        seed = 10_000 + case
        key = synth.make_key(kb, seed=seed)
        data = synth.make_pages(n, pb, seed=seed + 1)
        ivs = synth.make_ivs(n, seed=seed + 2) if mode == 0 else None
        exp = oracle_pages(d, mode, key, data, n, pb, ivs)
        kg.set_host_path(hp, 1 << 20)
        try:
            got = gpu_pages(d, mode, key, data, n, pb, ivs, where=where, inplace=inplace)
        finally:
            kg.set_host_path(kg.HOST_AUTO, 32 << 20)
        assert first_mismatch(got, exp) is None, dict(case=case, d=d, mode=mode, kb=kb, n=n, pb=pb, where=where,
                                                      inplace=inplace, hp=hp)


def test_random_large_batches_sampled():
    """Large batches (CTA pools active) with random page sizes: every page at a
    CTA-range boundary plus random pages are checked against the oracle."""
    kg, torch = kg_ready()
    rng = np.random.default_rng(1305)
    for case in range(10):
        pb = 16 * int(rng.integers(1, 260))
        n = int(64 * 148 + rng.integers(0, 3000))
        if n * pb > (96 << 20):
            n = (96 << 20) // pb
        d = int(rng.integers(0, 2)) if pb * n < (16 << 20) else 1
        mode = int(rng.integers(0, 2))
        inplace = bool(rng.integers(0, 2))
        key = synth.make_key(16, seed=case)
        data = synth.make_pages(n, pb, seed=case + 100)
        ivs = synth.make_ivs(n, seed=case + 200) if mode == 0 else None
        got = gpu_pages(d, mode, key, data, n, pb, ivs, where="device", inplace=inplace)
        pages = set(rng.integers(0, n, 40).tolist())
        for c in range(149):
            b = (n * c) // 148
            pages |= {max(0, b - 1), min(n - 1, b)}
        for p in sorted(pages):
            sl = slice(p * pb, (p + 1) * pb)
            iv = None if ivs is None else ivs[16 * p:16 * p + 16]
            exp = oracle_pages(d, mode, key, data[sl], 1, pb, iv)
            assert np.array_equal(got[sl], exp), dict(case=case, pb=pb, n=n, d=d, mode=mode, inplace=inplace, page=p)
