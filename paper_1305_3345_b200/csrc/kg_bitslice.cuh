// kg_bitslice.cuh -- bitsliced AES inverse cipher on 32 blocks per thread, for
// the bitsliced warps of the hybrid decryption kernel (kg_kernels.cu,
// kg_hybrid).  Included by kg_kernels.cu only.
//
// Why (profiles/r2_bitslice): the T-table round saturates the
// SM's shared-memory data path (16 lookups per block-round) while using ~75%
// of the ALU pipe.  Two warps running this ALU-only (LOP3) formulation on two
// of the four SM sub-partitions add ~0.16 block-rounds/clk/SM while the other
// 14 T-table warps keep the lookup pipe saturated: 2.12 vs 1.99 block-rounds
// per clock per SM in isolation.
//
// State layout (one thread): s[(c*4 + r)*8 + b] holds bit b of state byte
// (row r, column c) -- FIPS-197 §3.4 byte 4c + r -- of 32 blocks, block k in
// bit k.  A block's little-endian 32-bit word c is state column c, so word
// bit i is plane c*32 + i: the bit-matrix transpose below maps 32 blocks'
// words c straight onto planes c*32 .. c*32+31.
//
// The round follows FIPS-197 §5.3 (InvCipher) step by step:
//   InvShiftRows (register renaming), InvSubBytes (kg_bs_inv_sbox.cuh: the
//   inverse S-box circuit generated around the Boyar-Peralta nonlinear core,
//   verified on all 256 inputs), AddRoundKey (128 masks, 0 or ~0 per bit),
//   InvMixColumns (as MixColumns after the {04}-multiple pre-step, folded into
//   the output XORs; see bs_inv_mix).
#pragma once
#include <stdint.h>

#include "kg_bs_inv_sbox.cuh"

namespace kg {
namespace bs {

__device__ __forceinline__ void xtime8(const uint32_t *a, uint32_t *o) {
    // {02}*a on 8 bit-planes (a[0] = LSB): shift up, reduce by x^8 = x^4+x^3+x+1
    o[0] = a[7];
    o[1] = a[0] ^ a[7];
    o[2] = a[1];
    o[3] = a[2] ^ a[7];
    o[4] = a[3] ^ a[7];
    o[5] = a[4];
    o[6] = a[5];
    o[7] = a[6];
}

// Pin 8 values at this point of the volatile-ordered schedule.  S-boxes
// bracketed by pins are evaluated one after another: ptxas otherwise
// interleaves several of them and spills (profiles/r2_bitslice).
__device__ __forceinline__ void pin8(uint32_t *x) {
    asm volatile("" : "+r"(x[0]), "+r"(x[1]), "+r"(x[2]), "+r"(x[3]), "+r"(x[4]), "+r"(x[5]), "+r"(x[6]), "+r"(x[7]));
}

// In-place 32x32 bit-matrix transpose: afterwards bit k of a[i] is the old
// bit i of a[k] (its own inverse).  Five swap stages of 16 word pairs.
__device__ __forceinline__ void transpose32(uint32_t *a) {
    uint32_t m = 0x0000FFFFu;
#pragma unroll
    for (int j = 16; j != 0; j >>= 1, m ^= (m << j)) {
#pragma unroll
        for (int k = 0; k < 32; k++) {
            if (k & j) continue;
            const uint32_t t = ((a[k] >> j) ^ a[k + j]) & m;
            a[k + j] ^= t;
            a[k] ^= t << j;
        }
    }
}

// InvShiftRows + InvSubBytes + AddRoundKey(k) on s -> t (FIPS-197 §5.3.1,
// §5.3.2, §5.1.4).  InvSubBytes works on single bytes, so it commutes with
// the byte permutation InvShiftRows: S-boxes first, in place, then the
// permutation is a renaming.  k: 128 masks in shared memory (uniform address:
// one broadcast wavefront per LDS.128).
__device__ __forceinline__ void inv_sub_shift_key(uint32_t *s, uint32_t *t, const uint4 *k) {
#pragma unroll
    for (int byte = 0; byte < 16; byte++) {
        pin8(s + 8 * byte);
        bs_inv_sbox_bp(s + 8 * byte);
        pin8(s + 8 * byte);
    }
    // row r of column c comes from column c - r (§5.3.1: s'[r][c] = s[r][c - r mod 4])
#pragma unroll
    for (int c = 0; c < 4; c++)
#pragma unroll
        for (int r = 0; r < 4; r++)
#pragma unroll
            for (int q = 0; q < 2; q++) {
                const uint4 kk = k[((c * 4 + r) * 8 + 4 * q) / 4];
                const int d = (c * 4 + r) * 8 + 4 * q, src = (((c - r + 4) & 3) * 4 + r) * 8 + 4 * q;
                t[d + 0] = s[src + 0] ^ kk.x;
                t[d + 1] = s[src + 1] ^ kk.y;
                t[d + 2] = s[src + 2] ^ kk.z;
                t[d + 3] = s[src + 3] ^ kk.w;
            }
}

// InvMixColumns (FIPS-197 §5.3.3) of t -> s.  With a_r the column's bytes,
// U = {04}(a0 ^ a2), V = {04}(a1 ^ a3) and e_r = a_r ^ (r even ? U : V):
// InvMixColumns(a) = MixColumns(e) (the {0e},{0b},{0d},{09} matrix is the
// {02},{03},{01},{01} one times the {05},{00},{04},{00} one).  The e sum is
// the a sum T and e_r ^ e_{r+1} = a_r ^ a_{r+1} ^ U ^ V, so
//   out_r = a_r ^ {02}(a_r ^ a_{r+1}) ^ T ^ {02}(U ^ V) ^ (r even ? U : V).
__device__ __forceinline__ void inv_mix(const uint32_t *t, uint32_t *s) {
#pragma unroll
    for (int c = 0; c < 4; c++) {
        const uint32_t *a = t + c * 32;
        uint32_t TU[8], TV[8];
        {
            uint32_t u[8], x1[8], U[8], V[8], W[8];
#pragma unroll
            for (int b = 0; b < 8; b++) u[b] = a[b] ^ a[16 + b];
            xtime8(u, x1);
            xtime8(x1, U);
#pragma unroll
            for (int b = 0; b < 8; b++) u[b] = a[8 + b] ^ a[24 + b];
            xtime8(u, x1);
            xtime8(x1, V);
#pragma unroll
            for (int b = 0; b < 8; b++) u[b] = U[b] ^ V[b];
            xtime8(u, W);
#pragma unroll
            for (int b = 0; b < 8; b++) {
                const uint32_t T = a[b] ^ a[8 + b] ^ a[16 + b] ^ a[24 + b] ^ W[b];
                TU[b] = T ^ U[b];
                TV[b] = T ^ V[b];
            }
        }
#pragma unroll
        for (int r = 0; r < 4; r++) {
            uint32_t w[8], y2[8];
#pragma unroll
            for (int b = 0; b < 8; b++) w[b] = a[r * 8 + b] ^ a[((r + 1) & 3) * 8 + b];
            xtime8(w, y2);
#pragma unroll
            for (int b = 0; b < 8; b++) s[(c * 4 + r) * 8 + b] = a[r * 8 + b] ^ y2[b] ^ ((r & 1) ? TV[b] : TU[b]);
        }
    }
}

// FIPS-197 §5.3 InvCipher of the 32 blocks in s: AddRoundKey(Nr); Nr-1 rounds
// of InvShiftRows, InvSubBytes, AddRoundKey(r), InvMixColumns; the final
// InvShiftRows, InvSubBytes, AddRoundKey(0).  msk[r] = the 128 masks of round
// key w[4r .. 4r+3] of the (encryption) key schedule.
template <int NR>
__device__ __forceinline__ void inv_cipher(uint32_t *s, const uint4 (*msk)[32]) {
#pragma unroll
    for (int i = 0; i < 32; i++) {
        const uint4 kk = msk[NR][i];
        s[4 * i + 0] ^= kk.x;
        s[4 * i + 1] ^= kk.y;
        s[4 * i + 2] ^= kk.z;
        s[4 * i + 3] ^= kk.w;
    }
#pragma unroll 1
    for (int r = NR - 1; r >= 1; --r) {
        uint32_t t[128];
        inv_sub_shift_key(s, t, msk[r]);
        inv_mix(t, s);
    }
    uint32_t t[128];
    inv_sub_shift_key(s, t, msk[0]);
#pragma unroll
    for (int i = 0; i < 128; i++) s[i] = t[i];
}

}  // namespace bs
}  // namespace kg
