#!/usr/bin/env python
"""Generate the bitsliced AES S-box / inverse S-box circuits used by the
bitsliced kernel (paper_1305_3345_b200/csrc/kg_sbox_bs.cuh).

GPU-path code, independent of oracle/: the S-box is derived here from a
tower-field construction GF(((2^2)^2)^2) (polynomial bases w^2=w+1,
z^2=z+w, y^2=y+M), the field isomorphism to the AES polynomial basis
x^8+x^4+x^3+x+1 (FIPS-197 §4.2) found by searching for a root of that
polynomial in the tower field, and the affine map of FIPS-197 §5.1.1 as a
matrix.  The emitted straight-line code is verified exhaustively here against
an S-box computed by brute-force inversion (x^254) before it is written.

usage: python tools/gen_sbox_circuit.py > paper_1305_3345_b200/csrc/kg_sbox_bs.cuh
"""
import itertools
import sys

# ---- AES field GF(2^8) mod x^8+x^4+x^3+x+1 ----------------------------------


def aes_mul(a, b):
    p = 0
    for i in range(8):
        if (b >> i) & 1:
            p ^= a << i
    for bit in range(14, 7, -1):
        if (p >> bit) & 1:
            p ^= 0x11B << (bit - 8)
    return p


def aes_inv(a):
    r, e, base = 1, 254, a
    while e:
        if e & 1:
            r = aes_mul(r, base)
        base = aes_mul(base, base)
        e >>= 1
    return r if a else 0


def rotl8(x, s):
    return ((x << s) | (x >> (8 - s))) & 0xFF


def affine(b):
    return b ^ rotl8(b, 1) ^ rotl8(b, 2) ^ rotl8(b, 3) ^ rotl8(b, 4) ^ 0x63


SBOX = [affine(aes_inv(x)) for x in range(256)]
INV_SBOX = [0] * 256
for x, y in enumerate(SBOX):
    INV_SBOX[y] = x

# ---- tower field, elements as ints: GF4 2 bits (a1 a0), GF16 = (A1:GF4, A0:GF4) 4 bits,
# GF256 = (A1:GF16, A0:GF16) 8 bits --------------------------------------------


def g4_mul(a, b):
    a1, a0, b1, b0 = a >> 1, a & 1, b >> 1, b & 1
    hi = (a1 & b1) ^ (a1 & b0) ^ (a0 & b1)
    lo = (a1 & b1) ^ (a0 & b0)
    return (hi << 1) | lo


N4 = 0b10  # w


def g16_mul(a, b):
    a1, a0, b1, b0 = a >> 2, a & 3, b >> 2, b & 3
    t = g4_mul(a1, b1)
    hi = g4_mul(a1 ^ a0, b1 ^ b0) ^ g4_mul(a0, b0)
    lo = g4_mul(N4, t) ^ g4_mul(a0, b0)
    return (hi << 2) | lo


def g256_mul(a, b, M):
    a1, a0, b1, b0 = a >> 4, a & 15, b >> 4, b & 15
    t = g16_mul(a1, b1)
    hi = g16_mul(a1 ^ a0, b1 ^ b0) ^ g16_mul(a0, b0)
    lo = g16_mul(M, t) ^ g16_mul(a0, b0)
    return (hi << 4) | lo


def find_M():
    for M in range(1, 16):
        # y^2 + y + M irreducible over GF(16): no root
        if all(g16_mul(y, y) ^ y ^ M for y in range(16)):
            return M
    raise RuntimeError


M16 = find_M()


def t_pow(t, e):
    r = 1
    for _ in range(e):
        r = g256_mul(r, t, M16)
    return r


def find_iso():
    for t in range(2, 256):
        # root of x^8+x^4+x^3+x+1 in the tower field
        v = t_pow(t, 8) ^ t_pow(t, 4) ^ t_pow(t, 3) ^ t ^ 1
        if v == 0:
            cols = [t_pow(t, i) for i in range(8)]  # image of AES basis element x^i
            return cols
    raise RuntimeError


ISO = find_iso()


def mat_apply(cols, v):
    r = 0
    for i in range(8):
        if (v >> i) & 1:
            r ^= cols[i]
    return r


def mat_inverse(cols):
    # columns -> solve by brute force (256 elements)
    table = {mat_apply(cols, v): v for v in range(256)}
    assert len(table) == 256
    return [table[1 << i] for i in range(8)]


ISO_INV = mat_inverse(ISO)


def aff_cols():
    return [affine(1 << i) ^ 0x63 for i in range(8)]


AFF = aff_cols()
AFF_INV = mat_inverse(AFF)


def compose(A, B):  # A after B
    return [mat_apply(A, B[i]) for i in range(8)]


# S(x)   = AFF( ISO_INV( inv_t( ISO(x) ) ) ) ^ 0x63
# InvS(x)= ISO_INV( inv_t( ISO( AFF_INV(x ^ 0x63) ) ) )
S_IN = ISO
S_OUT = compose(AFF, ISO_INV)
S_OUT_C = 0x63
IS_IN = compose(ISO, AFF_INV)
IS_IN_C = mat_apply(compose(ISO, AFF_INV), 0x63)
IS_OUT = ISO_INV


def inv_tower(a):
    # GF(256) = GF(16)[y]/(y^2+y+M):  d = a0^2 + a0 a1 + M a1^2 ; inv = d^-1 (a1 y + (a0+a1))
    a1, a0 = a >> 4, a & 15
    d = g16_mul(a0, a0) ^ g16_mul(a0, a1) ^ g16_mul(M16, g16_mul(a1, a1))
    di = [x for x in range(16) if g16_mul(d, x) == 1]
    di = di[0] if di else 0
    return (g16_mul(di, a1) << 4) | g16_mul(di, a0 ^ a1)


assert all(mat_apply(S_OUT, inv_tower(mat_apply(S_IN, x))) ^ S_OUT_C == SBOX[x] for x in range(256))
assert all(mat_apply(IS_OUT, inv_tower(mat_apply(IS_IN, x) ^ IS_IN_C)) == INV_SBOX[x] for x in range(256))

# ---- circuit emission: symbolic straight-line code over 32-bit slices ------------


class Gen:
    def __init__(self):
        self.lines = []
        self.n = 0

    def tmp(self, expr):
        name = f"t{self.n}"
        self.n += 1
        self.lines.append(f"    const uint32_t {name} = {expr};")
        return name

    # GF(2) ops on names
    def x(self, a, b):
        return self.tmp(f"{a} ^ {b}")

    def a(self, a, b):
        return self.tmp(f"{a} & {b}")

    # GF4 values: (hi, lo)
    def g4_mul(self, p, q):
        a1, a0 = p
        b1, b0 = q
        # Karatsuba: hi = (a1^a0)(b1^b0) ^ a0b0 ; lo = a1b1 ^ a0b0
        m11 = self.a(a1, b1)
        m00 = self.a(a0, b0)
        mss = self.a(self.x(a1, a0), self.x(b1, b0))
        return (self.x(mss, m00), self.x(m11, m00))

    def g4_add(self, p, q):
        return (self.x(p[0], q[0]), self.x(p[1], q[1]))

    def g4_sq(self, p):  # (a1 w + a0)^2 = a1 w + (a1 + a0)
        return (p[0], self.x(p[0], p[1]))

    def g4_mulw(self, p):  # * w: hi = a1 + a0, lo = a1
        return (self.x(p[0], p[1]), p[0])

    def g4_sq_mulw(self, p):  # w * p^2 : p^2 = (a1, a1^a0); *w -> (a1 ^ a1 ^ a0, a1) = (a0, a1)
        return (p[1], p[0])

    # GF16 values: (A1, A0) of GF4
    def g16_mul(self, P, Q):
        A1, A0 = P
        B1, B0 = Q
        t11 = self.g4_mul(A1, B1)
        t00 = self.g4_mul(A0, B0)
        tss = self.g4_mul(self.g4_add(A1, A0), self.g4_add(B1, B0))
        hi = self.g4_add(tss, t00)
        lo = self.g4_add(self.g4_mulw(t11), t00)
        return (hi, lo)

    def g16_add(self, P, Q):
        return (self.g4_add(P[0], Q[0]), self.g4_add(P[1], Q[1]))

    def g16_sq(self, P):
        # (A1 z + A0)^2 = A1^2 z^2 + A0^2 = A1^2 z + (A1^2 w + A0^2)
        A1, A0 = P
        s1 = self.g4_sq(A1)
        s0 = self.g4_sq(A0)
        return (s1, self.g4_add(self.g4_mulw(s1), s0))

    def g16_mulconst(self, c, P):
        # multiply by the constant c (int) via its linear map, emitted as XORs
        bits = [P[1][1], P[1][0], P[0][1], P[0][0]]  # bit0..bit3 = A0.lo, A0.hi, A1.lo, A1.hi
        cols = [g16_mul(c, 1 << i) for i in range(4)]
        out = []
        for ob in range(4):
            terms = [bits[i] for i in range(4) if (cols[i] >> ob) & 1]
            acc = terms[0] if terms else "0u"
            for t in terms[1:]:
                acc = self.x(acc, t)
            out.append(acc)
        return ((out[3], out[2]), (out[1], out[0]))

    def g16_inv(self, P):
        # d = A0^2 + A0 A1 + N A1^2 ; inv = d^-1 (A1 z + (A0 + A1)); GF4 inverse = square
        A1, A0 = P
        d = self.g4_add(self.g4_add(self.g4_sq(A0), self.g4_mul(A0, A1)), self.g4_sq_mulw(A1))
        di = self.g4_sq(d)
        return (self.g4_mul(di, A1), self.g4_mul(di, self.g4_add(A0, A1)))

    def g256_inv(self, P):
        A1, A0 = P
        d = self.g16_add(self.g16_add(self.g16_sq(A0), self.g16_mul(A0, A1)),
                         self.g16_mulconst(M16, self.g16_sq(A1)))
        di = self.g16_inv(d)
        return (self.g16_mul(di, A1), self.g16_mul(di, self.g16_add(A0, A1)))

    def matvec(self, cols, ins, const=0):
        outs = []
        for ob in range(8):
            terms = [ins[i] for i in range(8) if (cols[i] >> ob) & 1]
            acc = terms[0] if terms else "0u"
            for t in terms[1:]:
                acc = self.x(acc, t)
            if (const >> ob) & 1:
                acc = self.tmp(f"~{acc}")
            outs.append(acc)
        return outs


def to_tower(bits):  # bit list (bit0..7) -> nested tuple
    return (((bits[7], bits[6]), (bits[5], bits[4])), ((bits[3], bits[2]), (bits[1], bits[0])))


def from_tower(T):
    ((a, b), (c, d)), ((e, f), (g, h)) = T
    return [h, g, f, e, d, c, b, a]


def emit(name, cin, cconst, cout, coutconst):
    G = Gen()
    ins = [f"x[{i}]" for i in range(8)]
    y = G.matvec(cin, ins, cconst)
    z = from_tower(G.g256_inv(to_tower(y)))
    o = G.matvec(cout, z, coutconst)
    body = "\n".join(G.lines)
    assigns = "\n".join(f"    x[{i}] = {o[i]};" for i in range(8))
    code = (f"// {name}: {len([l for l in G.lines])} straight-line ops before ptxas LOP3 fusion\n"
            f"__device__ __forceinline__ void {name}(uint32_t x[8]) {{\n{body}\n{assigns}\n}}\n")
    # verify by simulation over all 256 inputs in parallel (bit j of each slice = input j)
    env = {}
    for i in range(8):
        v = 0
        for inp in range(256):
            if (inp >> i) & 1:
                v |= 1 << inp
        env[f"x[{i}]"] = v
    mask = (1 << 256) - 1
    import re
    for line in G.lines:
        m = re.match(r"\s*const uint32_t (t\d+) = (.*);", line)
        nm, expr = m.group(1), m.group(2)
        e = expr
        if e.startswith("~"):
            val = (~env[e[1:]]) & mask
        elif " ^ " in e:
            a, b = e.split(" ^ ")
            val = env.get(a, 0) ^ env.get(b, 0)
        elif " & " in e:
            a, b = e.split(" & ")
            val = env[a] & env[b]
        else:
            raise ValueError(e)
        env[nm] = val
    outs = [env[o[i]] if o[i] != "0u" else 0 for i in range(8)]
    return code, outs


s_code, s_out = emit("bs_sbox", S_IN, 0, S_OUT, S_OUT_C)
is_code, is_out = emit("bs_inv_sbox", IS_IN, IS_IN_C, IS_OUT, 0)
for inp in range(256):
    got = sum(((s_out[i] >> inp) & 1) << i for i in range(8))
    assert got == SBOX[inp], (inp, got, SBOX[inp])
    got = sum(((is_out[i] >> inp) & 1) << i for i in range(8))
    assert got == INV_SBOX[inp], (inp, got, INV_SBOX[inp])

print(f"""// kg_sbox_bs.cuh -- GENERATED by tools/gen_sbox_circuit.py; do not edit.
// Bitsliced AES S-box / inverse S-box over 8 slices (x[i] = bit i of 32
// bytes in parallel), via GF(((2^2)^2)^2) tower-field inversion (w^2=w+1,
// z^2=z+w, y^2=y+{M16:#x}) between the FIPS-197 §4.2 field isomorphism and
// the §5.1.1 affine map.  Verified exhaustively by the generator.
#pragma once
#include <stdint.h>

{s_code}
{is_code}""")
