"""Pins of the C oracle against values fixed by FIPS-197 and SP 800-38A
(tests/golden/*, each file citing its source), plus exhaustive identities.
None of these re-types the oracle's own formulas."""
import os
import subprocess

import numpy as np
import pytest

import oracle
from conftest import GOLDEN, ROOT


def h(s):
    return bytes.fromhex(s)


def test_c_kat_binary():
    exe = os.path.join(ROOT, "build", "test_kat")
    os.makedirs(os.path.dirname(exe), exist_ok=True)
    src = [os.path.join(ROOT, "oracle", f) for f in ("kgo_aes.c", "kgo_pages.c", "test_kat.c")]
    subprocess.check_call(["gcc", "-std=c99", "-O2", "-D_POSIX_C_SOURCE=200809L", "-o", exe] + src + ["-lpthread"])
    out = subprocess.run([exe, GOLDEN], capture_output=True, text=True)
    assert out.returncode == 0, out.stderr + out.stdout
    assert "0 failures" in out.stdout


def test_gf_and_sbox_spot_values(golden):
    for row in golden("gf_sbox.txt"):
        kind, args, exp = row[0], [int(x, 16) for x in row[1:-1]], int(row[-1], 16)
        if kind == "mul":
            assert oracle.gf_mul(*args) == exp, row
            assert oracle.gf_mul(args[1], args[0]) == exp, row
        elif kind == "sbox":
            assert oracle.sbox(args[0]) == exp, row
        elif kind == "isbox":
            assert oracle.inv_sbox(args[0]) == exp, row


def test_sbox_is_permutation_and_inverse():
    s = [oracle.sbox(x) for x in range(256)]
    assert sorted(s) == list(range(256))
    assert all(oracle.inv_sbox(oracle.sbox(x)) == x for x in range(256))
    # FIPS-197 §5.1.1: the S-box has no fixed points and no "opposite" fixed points
    assert all(s[x] != x and s[x] != (x ^ 0xFF) for x in range(256))


def test_gf_field_axioms_exhaustive():
    # every non-zero element has exactly one inverse; {01} is the identity; xtime = •{02}
    for a in range(256):
        assert oracle.gf_mul(a, 1) == a
        assert oracle.xtime(a) == oracle.gf_mul(a, 2)
        if a:
            inv = [b for b in range(1, 256) if oracle.gf_mul(a, b) == 1]
            assert len(inv) == 1


def test_key_expansion_appendix_a(golden):
    for keyh, i, wi in golden("fips197_appA_keyexp.txt"):
        nr, w = oracle.key_expansion(h(keyh))
        i = int(i)
        assert w[4 * i:4 * i + 4] == h(wi), (keyh[:8], i)
    assert oracle.key_expansion(bytes(16))[0] == 10
    assert oracle.key_expansion(bytes(24))[0] == 12
    assert oracle.key_expansion(bytes(32))[0] == 14
    with pytest.raises(ValueError):
        oracle.key_expansion(bytes(20))


def test_appendix_b_round_trace(golden):
    """Every step transformation separately against FIPS-197 Appendix B."""
    rows = {(int(r), s): h(v) for r, s, v in golden("fips197_appB_trace.txt")}
    key = h("2b7e151628aed2a6abf7158809cf4f3c")
    nr, w = oracle.key_expansion(key)
    pt = h("3243f6a8885a308d313198a2e0370734")
    assert oracle.add_round_key(pt, w[0:16]) == rows[(1, "start")]
    assert oracle.step("sub_bytes", rows[(1, "start")]) == rows[(1, "sub")]
    assert oracle.step("shift_rows", rows[(1, "sub")]) == rows[(1, "shift")]
    assert oracle.step("mix_columns", rows[(1, "shift")]) == rows[(1, "mix")]
    assert w[16:32] == rows[(1, "rk")]
    assert oracle.add_round_key(rows[(1, "mix")], rows[(1, "rk")]) == rows[(2, "start")]
    assert oracle.step("sub_bytes", rows[(10, "start")]) == rows[(10, "sub")]
    assert oracle.step("shift_rows", rows[(10, "sub")]) == rows[(10, "shift")]
    assert w[160:176] == rows[(10, "rk")]
    assert oracle.add_round_key(rows[(10, "shift")], rows[(10, "rk")]) == rows[(11, "out")]
    # inverse steps undo the forward ones
    for name in ("sub_bytes", "shift_rows", "mix_columns"):
        x = rows[(1, "start")]
        assert oracle.step("inv_" + name, oracle.step(name, x)) == x


def test_mix_columns_examples(golden):
    for inp, exp in golden("mixcolumns.txt"):
        st = h(inp) * 4
        assert oracle.step("mix_columns", st) == h(exp) * 4
        assert oracle.step("inv_mix_columns", h(exp) * 4) == st


def test_cipher_kats(golden):
    for label, k, p, c in golden("fips197_cipher_kat.txt"):
        assert oracle.cipher(h(k), h(p)) == h(c), label
        assert oracle.inv_cipher(h(k), h(c)) == h(p), label


def test_cbc_sp800_38a(golden):
    for label, k, iv, p, c in golden("sp800_38a_cbc.txt"):
        got = oracle.pages(oracle.ENCRYPT, oracle.MODE_CBC, h(k), h(p), 1, 64, h(iv))
        assert got.tobytes() == h(c), label
        got = oracle.pages(oracle.DECRYPT, oracle.MODE_CBC, h(k), h(c), 1, 64, h(iv))
        assert got.tobytes() == h(p), label
        # the same chain split as 4 one-block pages whose IVs are the previous
        # ciphertext blocks (SP 800-38A §6.2: C_{j-1} plays the IV's role)
        ivs = h(iv) + h(c)[:48]
        got = oracle.pages(oracle.ENCRYPT, oracle.MODE_CBC, h(k), h(p), 4, 16, ivs)
        assert got.tobytes() == h(c), label


def test_page16_zero_iv_is_ecb(golden):
    """Identity (i): page_bytes=16 with IV=0 is single-block ECB = FIPS-197 App. C."""
    for label, k, p, c in golden("fips197_cipher_kat.txt"):
        got = oracle.pages(oracle.ENCRYPT, oracle.MODE_CBC, h(k), h(p), 1, 16, bytes(16))
        assert got.tobytes() == h(c), label
        got = oracle.pages(oracle.DECRYPT, oracle.MODE_ECB, h(k), h(c), 1, 16, None)
        assert got.tobytes() == h(p), label


def test_bad_arguments_rejected():
    with pytest.raises(ValueError):
        oracle.pages(0, 0, bytes(16), bytes(15), 1, 15, bytes(16))
    with pytest.raises(ValueError):
        oracle.pages(0, 0, bytes(17), bytes(16), 1, 16, bytes(16))
    with pytest.raises(ValueError):
        oracle.pages(2, 0, bytes(16), bytes(16), 1, 16, bytes(16))
