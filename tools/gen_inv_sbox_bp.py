#!/usr/bin/env python
"""Emit tools/kg_inv_sbox_bp.cuh: the AES INVERSE S-box as a bitsliced circuit
built around the Boyar-Peralta nonlinear core (the same 34-AND middle section
as tools/gen_sbox_bp.py's forward circuit), for the bitsliced / hybrid
decryption measurement (tools/hybrid_throttle.cu).

InvS(y) = Inv(A^-1 (y ^ 0x63)) (FIPS-197 §5.3.2), where Inv is inversion in
GF(2^8) and A the S-box's affine matrix.  The BP circuit computes
S(x) = A Inv(x) ^ 0x63 as  top (linear in x) -> middle (nonlinear, shared) ->
bottom (linear in the 18 products M46..M63, NOTs for 0x63).  So the inverse
circuit is
  * top'    : the forward top-layer signals evaluated at x = A^-1 (y ^ 0x63),
              i.e. AFFINE functions of y (coefficients found by evaluating on
              0 and the unit vectors);
  * middle  : unchanged;
  * bottom' : A^-1 applied to the forward bottom layer without its NOTs,
              i.e. Inv(x) as LINEAR functions of M46..M63;
and both linear layers are emitted as XOR networks found by Paar's greedy
common-subexpression heuristic.  The circuit is evaluated on all 256 inputs
against the inverse S-box computed here from its definition before anything
is written.  Tool code: not the product library, not the oracle.

usage: python tools/gen_inv_sbox_bp.py [OUT.cuh]   (default: stdout, named kg_inv_sbox_bp.cuh)
  tools/kg_inv_sbox_bp.cuh -- the hybrid microbenchmark's copy (the product kernel that used
  it, kg_hybrid, is in git history: profiles/r2_hybrid)
"""
import os
import sys

sys.path.insert(0, __import__("os").path.dirname(__file__))
import gen_sbox_bp as fwd  # noqa: E402  (CIRCUIT text, S-box from its definition)

LINES = fwd.LINES
TOP = [l for l in LINES if l.split("=")[0].strip().startswith("T")]
MID = [l for l in LINES if l.split("=")[0].strip().startswith("M")]
BOT = [l for l in LINES if l.split("=")[0].strip()[0] in "LS"]


def affine_a(b):
    r = lambda x, s: ((x << s) | (x >> (8 - s))) & 0xFF  # noqa: E731
    return b ^ r(b, 1) ^ r(b, 2) ^ r(b, 3) ^ r(b, 4)


A_INV = [0] * 256
for v in range(256):
    A_INV[affine_a(v)] = v
INV_SBOX = [0] * 256
for x in range(256):
    INV_SBOX[fwd.SBOX[x]] = x


def top_signals(x):
    """forward top-layer signals (T1..T27 and U0..U7) for input byte x"""
    env = {f"U{i}": (x >> (7 - i)) & 1 for i in range(8)}
    for l in TOP:
        k, e = l.split("=", 1)
        env[k.strip()] = eval(e, {}, env) & 1
    return env


# ---- top': each signal the middle section reads, as an affine function of y
mid_inputs = sorted({tok for l in MID for tok in l.replace("=", " ").replace("^", " ").replace("&", " ").split()
                     if tok[0] in "TU"}, key=lambda s: (s[0], int(s[1:])))
sig0 = top_signals(A_INV[0 ^ 0x63])
top_aff = {}
for s in mid_inputs:
    const = sig0[s]
    mask = 0
    for k in range(8):  # y bit k (k = 0: MSB, as the circuit's U0)
        y = 1 << (7 - k)
        if top_signals(A_INV[y ^ 0x63])[s] ^ const:
            mask |= 1 << k
    top_aff[s] = (mask, const)
# check affinity on all inputs
for y in range(256):
    sg = top_signals(A_INV[y ^ 0x63])
    for s, (mask, c) in top_aff.items():
        v = c
        for k in range(8):
            if mask >> k & 1:
                v ^= (y >> (7 - k)) & 1
        assert v == sg[s], (s, y)

# ---- bottom': Inv(x) bits as linear functions of the 18 products
prods = sorted({tok for l in BOT for tok in l.replace("=", " ").replace("^", " ").replace("~", " ")
                .replace("(", " ").replace(")", " ").split() if tok.startswith("M")}, key=lambda s: int(s[1:]))
assert len(prods) == 18
sym = {p: 1 << i for i, p in enumerate(prods)}
for l in BOT:
    k, e = [t.strip() for t in l.split("=", 1)]
    e = e.replace("~", "").replace("(", "").replace(")", "")
    v = 0
    for tok in e.split("^"):
        v ^= sym[tok.strip()]
    sym[k] = v
# S bit i (S0 = MSB) without the NOTs = (A Inv(x)) bit i; Inv(x) = A^-1 (that)
s_masks = [sym[f"S{i}"] for i in range(8)]  # masks over prods, MSB first
inv_masks = []
for i in range(8):  # output bit i (MSB first) of A^-1 z = XOR of z bits j where A^-1 has a 1
    m = 0
    for j in range(8):
        # column j of A^-1: A^-1 applied to unit vector with bit (7-j)
        col = A_INV[1 << (7 - j)]
        if (col >> (7 - i)) & 1:
            m ^= s_masks[j]
    inv_masks.append(m)


def paar(targets, n_in, names, prefix):
    """Paar's greedy XOR network: targets = list of bitmasks over n_in inputs.
    Returns (gate lines, output expressions)."""
    cols = [list(names)]  # signal names
    vecs = [1 << i for i in range(n_in)]  # each signal's mask over the original inputs
    rows = [set(i for i in range(n_in) if t >> i & 1) for t in targets]
    lines = []
    g = 0
    while True:
        best, cnt = None, 1
        n = len(vecs)
        counts = {}
        for r in rows:
            rl = sorted(r)
            for a in range(len(rl)):
                for b in range(a + 1, len(rl)):
                    counts[(rl[a], rl[b])] = counts.get((rl[a], rl[b]), 0) + 1
        for pair, c in counts.items():
            if c > cnt:
                best, cnt = pair, c
        if best is None:
            break
        a, b = best
        name = f"{prefix}{g}"
        g += 1
        lines.append(f"{name} = {cols[0][a]} ^ {cols[0][b]}")
        cols[0].append(name)
        vecs.append(vecs[a] ^ vecs[b])
        idx = len(vecs) - 1
        for r in rows:
            if a in r and b in r:
                r.discard(a)
                r.discard(b)
                r.add(idx)
    outs = []
    for r in rows:
        terms = [cols[0][i] for i in sorted(r)]
        outs.append(terms)
    return lines, outs


def main():
    ynames = [f"Y{k}" for k in range(8)]
    top_lines, top_outs = paar([top_aff[s][0] for s in mid_inputs], 8, ynames, "P")
    circuit = list(top_lines)
    n_top = len(top_lines)
    for s, terms in zip(mid_inputs, top_outs):
        e = " ^ ".join(terms) if terms else "0"
        if top_aff[s][1]:
            e = f"~({e})"
        circuit.append(f"{s} = {e}")
        n_top += max(0, len(terms) - 1) + (1 if top_aff[s][1] and len(terms) <= 1 else 0)
    circuit += MID
    bot_lines, bot_outs = paar(inv_masks, 18, prods, "Q")
    circuit += bot_lines
    for i, terms in enumerate(bot_outs):
        circuit.append(f"O{i} = {' ^ '.join(terms)}")

    def evaluate(y):
        env = {f"Y{k}": (y >> (7 - k)) & 1 for k in range(8)}
        for l in circuit:
            k, e = l.split("=", 1)
            env[k.strip()] = eval(e, {}, env) & 1
        return sum(env[f"O{i}"] << (7 - i) for i in range(8))

    bad = [y for y in range(256) if evaluate(y) != INV_SBOX[y]]
    if bad:
        sys.exit(f"inverse circuit wrong on {len(bad)} inputs, first {bad[0]:#04x}")
    gates = sum(max(1, l.count("^") + l.count("&")) for l in circuit if "=" in l)
    n_and = sum(l.count("&") for l in circuit)
    path = sys.argv[1] if len(sys.argv) > 1 else None
    fname = os.path.basename(path) if path else "kg_inv_sbox_bp.cuh"
    out = [f"// {fname} -- GENERATED by tools/gen_inv_sbox_bp.py; do not edit.",
           "// AES inverse S-box, bitsliced on 32 blocks per word: affine top layer (Paar XOR network),",
           "// the Boyar-Peralta nonlinear core (%d AND), linear bottom layer (Paar); ~%d two-input" % (n_and, gates),
           "// gates; verified on all 256 inputs at generation time.",
           "#pragma once",
           "#include <stdint.h>",
           "__device__ __forceinline__ void bs_inv_sbox_bp(uint32_t x[8]) {"]
    for k in range(8):
        out.append(f"    const uint32_t Y{k} = x[{7 - k}];")
    for l in circuit:
        k, e = [t.strip() for t in l.split("=", 1)]
        out.append(f"    const uint32_t {k} = {e};")
    for i in range(8):
        out.append(f"    x[{7 - i}] = O{i};")
    out.append("}")
    text = "\n".join(out) + "\n"
    if path:
        with open(path, "w") as f:
            f.write(text)
    else:
        sys.stdout.write(text)
    print(f"inverse S-box circuit: {gates} gates ({n_and} AND), top {len(top_lines)} shared XOR, "
          f"bottom {len(bot_lines)} shared XOR; verified on 256 inputs", file=sys.stderr)


if __name__ == "__main__":
    main()
