"""Parity of the hybrid decryption kernel (T-table warps + bitsliced warps,
kg_kernels.cu `kg_hybrid`) with the oracle, every byte.

The hybrid kernel runs for large device-input CBC/ECB decryption batches of
power-of-two pages (32 B .. 16 KiB) with at least 256 x (4096 / page_bytes)
... precisely: >= 32,768 block pairs per CTA.  Sizes here are ragged against
the 148-CTA grid, the 1,024-block bitsliced unit and the T-table pool, and
each test asserts that the hybrid kernel actually launched."""
import numpy as np
import pytest

import synth
from gpu_util import first_mismatch, gpu_pages, kg_ready, oracle_pages

pytestmark = pytest.mark.gpu


def run_hybrid(direction, mode, key_bytes, n, pb, inplace=False, seed=0):
    kg, _ = kg_ready()
    key = synth.make_key(key_bytes, seed=seed + 1)
    data = synth.make_pages(n, pb, seed=seed + 2)
    ivs = synth.make_ivs(n, seed=seed + 3) if mode == 0 else None
    h0 = kg.hybrid_launch_count()
    got = gpu_pages(direction, mode, key, data, n, pb, ivs, where="device", inplace=inplace)
    launched = kg.hybrid_launch_count() - h0
    exp = oracle_pages(direction, mode, key, data, n, pb, ivs)
    return got, exp, launched


@pytest.mark.parametrize("key_bytes", [16, 24, 32])
@pytest.mark.parametrize("mode", [0, 1])
def test_hybrid_4k_pages(mode, key_bytes):
    n = 40_009  # > 148 x 256 pages, ragged
    got, exp, launched = run_hybrid(1, mode, key_bytes, n, 4096, seed=10 * mode + key_bytes)
    assert launched == 1
    assert first_mismatch(got, exp) is None, f"first mismatch at byte {first_mismatch(got, exp)}"


@pytest.mark.parametrize("mode", [0, 1])
def test_hybrid_in_place(mode):
    n = 38_917
    got, exp, launched = run_hybrid(1, mode, 16, n, 4096, inplace=True, seed=300 + mode)
    assert launched == 1
    assert first_mismatch(got, exp) is None


@pytest.mark.parametrize("pb,n", [(32, 4_849_999), (1024, 160_001), (16384, 9_601), (256, 620_007)])
def test_hybrid_page_sizes(pb, n):
    got, exp, launched = run_hybrid(1, 0, 16, n, pb, seed=pb)
    assert launched == 1
    assert first_mismatch(got, exp) is None


def test_hybrid_off_is_not_used_for_small_batches():
    """Below the size floor the block-pair kernel runs (no hybrid launch)."""
    got, exp, launched = run_hybrid(1, 0, 16, 4_000, 4096, seed=77)
    assert launched == 0
    assert first_mismatch(got, exp) is None


def test_hybrid_matches_blockpair_kernel_on_c2():
    """The C2 batch (65,536 x 4 KiB, AES-128-CBC decrypt): hybrid output equals the
    oracle's; the same batch with the hybrid switched off in a child process
    (KG_HYBRID=0 is read once per process) is covered by test_fullsize_gpu."""
    got, exp, launched = run_hybrid(1, 0, 16, 65_536, 4096, seed=2)
    assert launched == 1
    assert np.array_equal(got, exp)
