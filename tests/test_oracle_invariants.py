"""CBC identities the oracle must satisfy (SURVEY.md §8c 'Page structure' and
'Invariants'): round trip, decrypt locality incl. the page boundary, encrypt
propagation, page-permutation equivariance, in-place == out-of-place, and
thread-count independence."""
import numpy as np

import oracle
import synth

N, PB = 6, 256
KEY = synth.make_key(16)


def data():
    return synth.make_pages(N, PB), synth.make_ivs(N)


def enc(x, ivs, key=KEY, n=N, pb=PB, **kw):
    return oracle.pages(0, 0, key, x, n, pb, ivs, **kw)


def dec(x, ivs, key=KEY, n=N, pb=PB, **kw):
    return oracle.pages(1, 0, key, x, n, pb, ivs, **kw)


def test_round_trip_all_key_sizes():
    p, iv = data()
    for kb in (16, 24, 32):
        k = synth.make_key(kb)
        assert np.array_equal(dec(enc(p, iv, k), iv, k), p)


def test_cbc_decrypt_identity_via_ecb():
    """P = ECB^-1(C) xor (IV || C_0..C_{m-2}) per page."""
    c, iv = data()
    p = dec(c, iv)
    e = oracle.pages(1, 1, KEY, c, N, PB, None)
    m = PB // 16
    for pg in range(N):
        cp = c[pg * PB:(pg + 1) * PB]
        prev = np.concatenate([iv[16 * pg:16 * pg + 16], cp[:PB - 16]])
        assert np.array_equal(p[pg * PB:(pg + 1) * PB], e[pg * PB:(pg + 1) * PB] ^ prev)
    assert m == 16


def test_decrypt_locality_and_page_boundary():
    c, iv = data()
    p = dec(c, iv)
    m = PB // 16
    for pg, j in [(0, 0), (2, 5), (3, m - 1)]:
        c2 = c.copy()
        byte = pg * PB + 16 * j + 3
        c2[byte] ^= 0x10
        p2 = dec(c2, iv)
        diff = np.nonzero(p != p2)[0]
        blk = diff // 16
        g = pg * m + j
        # block j changes (almost surely entirely), block j+1 exactly one bit, nothing else
        assert set(blk.tolist()) <= {g, g + 1}
        assert (p[g * 16:(g + 1) * 16] != p2[g * 16:(g + 1) * 16]).sum() >= 8
        if j + 1 < m:
            assert list(diff[blk == g + 1]) == [byte + 16]
            assert p2[byte + 16] ^ p[byte + 16] == 0x10
        else:
            # last block of the page: the next page is untouched
            assert g + 1 not in set(blk.tolist())


def test_encrypt_propagation():
    p, iv = data()
    c = enc(p, iv)
    m = PB // 16
    pg, j = 1, 3
    p2 = p.copy()
    p2[pg * PB + 16 * j] ^= 1
    c2 = enc(p2, iv)
    changed = sorted(set((np.nonzero(c != c2)[0] // 16).tolist()))
    assert changed == list(range(pg * m + j, (pg + 1) * m))


def test_iv_only_affects_own_page():
    p, iv = data()
    c = enc(p, iv)
    iv2 = iv.copy()
    iv2[16 * 4] ^= 0x80
    c2 = enc(p, iv2)
    pages_changed = sorted(set((np.nonzero(c != c2)[0] // PB).tolist()))
    assert pages_changed == [4]


def test_page_permutation_equivariance():
    p, iv = data()
    c = enc(p, iv)
    perm = np.array([3, 0, 5, 1, 4, 2])
    pp = p.reshape(N, PB)[perm].reshape(-1)
    ivp = iv.reshape(N, 16)[perm].reshape(-1)
    cp = enc(pp, ivp)
    assert np.array_equal(cp.reshape(N, PB), c.reshape(N, PB)[perm])


def test_in_place_and_threads():
    p, iv = data()
    c = enc(p, iv)
    x = c.copy()
    oracle.pages(1, 0, KEY, x, N, PB, iv, out=x)
    assert np.array_equal(x, p)
    for t in (1, 2, 3, 6, 16):
        assert np.array_equal(enc(p, iv, threads=t), c)
