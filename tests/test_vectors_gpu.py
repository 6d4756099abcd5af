"""Standard vectors through the C ABI on the GPU: SP 800-38A F.2.1-F.2.6 as
one 64-byte page; FIPS-197 App. B/C as a 16-byte page with IV = 0 (CBC) and
as ECB; the same vectors replicated across many pages/CTAs."""
import numpy as np
import pytest

from conftest import read_golden
from gpu_util import gpu_pages

pytestmark = pytest.mark.gpu
h = bytes.fromhex


def arr(b):
    return np.frombuffer(b, dtype=np.uint8).copy()


@pytest.mark.parametrize("where", ["device", "pinned"])
def test_sp800_38a_cbc(where):
    for label, k, iv, p, c in read_golden("sp800_38a_cbc.txt"):
        got = gpu_pages(0, 0, h(k), arr(h(p)), 1, 64, arr(h(iv)), where=where)
        assert got.tobytes() == h(c), label
        got = gpu_pages(1, 0, h(k), arr(h(c)), 1, 64, arr(h(iv)), where=where)
        assert got.tobytes() == h(p), label


def test_sp800_38a_replicated_over_many_pages():
    """5000 copies of the F.2 chain as 5000 pages: every page must decrypt alike
    (covers every CTA, warp and lane position)."""
    for label, k, iv, p, c in read_golden("sp800_38a_cbc.txt"):
        n = 5000
        got = gpu_pages(1, 0, h(k), arr(h(c) * n), n, 64, arr(h(iv) * n))
        assert got.tobytes() == h(p) * n, label
        got = gpu_pages(0, 0, h(k), arr(h(p) * n), n, 64, arr(h(iv) * n))
        assert got.tobytes() == h(c) * n, label


def test_fips197_blocks():
    for label, k, p, c in read_golden("fips197_cipher_kat.txt"):
        got = gpu_pages(0, 0, h(k), arr(h(p)), 1, 16, np.zeros(16, np.uint8))
        assert got.tobytes() == h(c), label
        got = gpu_pages(1, 0, h(k), arr(h(c)), 1, 16, np.zeros(16, np.uint8))
        assert got.tobytes() == h(p), label
        got = gpu_pages(0, 1, h(k), arr(h(p) * 333), 333, 16, None)
        assert got.tobytes() == h(c) * 333, label
        got = gpu_pages(1, 1, h(k), arr(h(c) * 64), 2, 512, None)
        assert got.tobytes() == h(p) * 64, label
