"""The oracle against an independent implementation (OpenSSL via the
`cryptography` package) on random jobs.  `cryptography` is used ONLY here,
to test the oracle; nothing in the product links or imports it."""
import numpy as np
import pytest

import oracle
import synth

cryptography = pytest.importorskip("cryptography")
from cryptography.hazmat.primitives.ciphers import Cipher, algorithms, modes  # noqa: E402


def openssl_cbc_pages(direction, key, data, n_pages, page_bytes, ivs):
    out = bytearray()
    for p in range(n_pages):
        c = Cipher(algorithms.AES(key), modes.CBC(ivs[16 * p:16 * p + 16]))
        ctx = c.encryptor() if direction == 0 else c.decryptor()
        out += ctx.update(data[p * page_bytes:(p + 1) * page_bytes]) + ctx.finalize()
    return bytes(out)


def openssl_ecb(direction, key, data):
    c = Cipher(algorithms.AES(key), modes.ECB())
    ctx = c.encryptor() if direction == 0 else c.decryptor()
    return ctx.update(data) + ctx.finalize()


def test_random_jobs_vs_openssl():
    rng = np.random.default_rng(1305)
    for job in range(300):
        kb = int(rng.choice([16, 24, 32]))
        n = int(rng.integers(1, 9))
        pb = 16 * int(rng.integers(1, 40))
        key = rng.integers(0, 256, kb, dtype=np.uint8).tobytes()
        data = rng.integers(0, 256, n * pb, dtype=np.uint8).tobytes()
        ivs = rng.integers(0, 256, 16 * n, dtype=np.uint8).tobytes()
        d = int(rng.integers(0, 2))
        got = oracle.pages(d, oracle.MODE_CBC, key, data, n, pb, ivs, threads=int(rng.integers(1, 4)))
        assert got.tobytes() == openssl_cbc_pages(d, key, data, n, pb, ivs), (job, kb, n, pb, d)
        got = oracle.pages(d, oracle.MODE_ECB, key, data, n, pb, None)
        assert got.tobytes() == openssl_ecb(d, key, data), (job, "ecb")


def test_seeded_4k_pages_vs_openssl():
    n = 64
    key = synth.make_key(32)
    data = synth.make_pages(n).tobytes()
    ivs = synth.make_ivs(n).tobytes()
    for d in (0, 1):
        got = oracle.pages(d, oracle.MODE_CBC, key, data, n, 4096, ivs, threads=4)
        assert got.tobytes() == openssl_cbc_pages(d, key, data, n, 4096, ivs)
