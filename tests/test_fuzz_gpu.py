"""Randomised parity sweep: random (direction, mode, key size, page count,
page size, residency, in-place, host path) cases, each compared byte for byte
with the oracle.  Sizes stay small so the oracle finishes quickly."""
import numpy as np
import pytest

import synth
from gpu_util import first_mismatch, gpu_pages, kg_ready, oracle_pages

pytestmark = pytest.mark.gpu


def test_random_cases():
    kg, torch = kg_ready()
    rng = np.random.default_rng(20261017)
    for case in range(150):
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
