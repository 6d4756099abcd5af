"""examples/kgpu_crypt.c end to end on the GPU: encrypt a file of 4 KiB pages
(+ a short tail page), compare every page with the oracle under the
example's IV scheme, then decrypt back to the original bytes."""
import os
import subprocess

import numpy as np
import pytest

import synth
from conftest import ROOT
from gpu_util import oracle_pages, torch_cuda

pytestmark = pytest.mark.gpu

FILE_IV = bytes([0x6b, 0x67, 0x70, 0x75, 0x2d, 0x62, 0x32, 0x30, 0x30, 0x2d, 0x65, 0x78, 0x61, 0x6d, 0x70, 0x6c])


def iv_of(p):
    return bytes(FILE_IV[b] ^ ((p >> (8 * b)) & 0xFF if b < 8 else 0) for b in range(16))


@pytest.mark.parametrize("key_bytes", [16, 32])
def test_kgpu_crypt_file(tmp_path, key_bytes):
    torch_cuda()
    exe = os.path.join(ROOT, "build", "kgpu_crypt")
    if not os.path.exists(exe):
        pytest.skip("build/kgpu_crypt not built")
    pages, tail = 37, 48
    data = synth.make_pages(1, pages * 4096 + tail, seed=key_bytes)
    key = synth.make_key(key_bytes, seed=99)
    src, enc, dec = tmp_path / "in", tmp_path / "enc", tmp_path / "dec"
    src.write_bytes(data.tobytes())
    subprocess.check_call([exe, "enc", key.hex(), str(src), str(enc)])
    subprocess.check_call([exe, "dec", key.hex(), str(enc), str(dec)])
    assert dec.read_bytes() == src.read_bytes()
    c = np.frombuffer(enc.read_bytes(), dtype=np.uint8)
    for p in list(range(pages)):
        exp = oracle_pages(0, 0, key, data[p * 4096:(p + 1) * 4096], 1, 4096, np.frombuffer(iv_of(p), np.uint8))
        assert np.array_equal(c[p * 4096:(p + 1) * 4096], exp), p
    exp = oracle_pages(0, 0, key, data[pages * 4096:], 1, tail, np.frombuffer(iv_of(pages), np.uint8))
    assert np.array_equal(c[pages * 4096:], exp)
