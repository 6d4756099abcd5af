// hybrid_throttle.cu -- can a rate-limited bitsliced warpgroup add throughput
// on top of T-table warps that saturate the LSU data pipe?
//
// profiles/r1_bitslice (tools/hybrid_bench.cu) measured 12 T-table warps + 4
// free-running bitsliced warps (tower-field S-box) at 1.872 block-rounds/clk/SM
// against 1.985 for T-table alone: the bitsliced warps' LOP3 stream took more
// ALU issue from the T-table warps (-0.41) than it added (+0.30).  The T-table
// round needs 24 ALU lane-ops per block-round against 16 LDS, so at the LSU
// bound (2 block-rounds/clk) it leaves 64 - 48 = 16 ALU lane-ops/clk/SM; the
// Boyar-Peralta bitsliced round needs ~63 per block-round, so the hybrid's
// ceiling is 2 + 16/63 = 2.25 (+13%) -- IF the bitsliced side takes only the
// ALU slots the T-table side leaves.  This benchmark rate-limits the
// bitsliced warps (__nanosleep after every S-box / every round, or fewer
// bitsliced warps) and reports both sides' block-rounds per SM clock.
//
// One 512-thread CTA per SM, 128 KiB of lane-replicated tables; every warp
// loops for 5 ms of %globaltimer.  Warpgroups 0-2: T-table rounds on two
// blocks per lane (the block-pair kernel's body shape).  Warpgroup 3:
// bitsliced AES-128 encryption rounds on 32 blocks per thread (BP S-box,
// ShiftRows by renaming, MixColumns, round-key masks in the constant bank),
// `setmaxnreg` 88 / 232.
//
// build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -Itools tools/hybrid_throttle.cu -o build/hybrid_throttle
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "kg_inv_sbox_bp.cuh"
#include "kg_sbox_bp.cuh"

__constant__ uint32_t c_rk[128];

__device__ __forceinline__ void xtime8(const uint32_t *a, uint32_t *o) {
    o[0] = a[7];
    o[1] = a[0] ^ a[7];
    o[2] = a[1];
    o[3] = a[2] ^ a[7];
    o[4] = a[3] ^ a[7];
    o[5] = a[4];
    o[6] = a[5];
    o[7] = a[6];
}

// SLEEP_SBOX: ns after every S-box (16 per round); SLEEP_ROUND: ns after every round
template <int SLEEP_SBOX>
__device__ __forceinline__ void bs_round(uint32_t *s) {
#pragma unroll
    for (int byte = 0; byte < 16; byte++) {
        bs_sbox_bp(s + 8 * byte);
        if (SLEEP_SBOX > 0) __nanosleep(SLEEP_SBOX);
    }
    uint32_t t[128];
#pragma unroll
    for (int c = 0; c < 4; c++)
#pragma unroll
        for (int r = 0; r < 4; r++)
#pragma unroll
            for (int b = 0; b < 8; b++) t[(c * 4 + r) * 8 + b] = s[(((c + r) & 3) * 4 + r) * 8 + b];
#pragma unroll
    for (int c = 0; c < 4; c++) {
        const uint32_t *a = t + c * 32;
        uint32_t T[8];
#pragma unroll
        for (int b = 0; b < 8; b++) T[b] = a[b] ^ a[8 + b] ^ a[16 + b] ^ a[24 + b];
#pragma unroll
        for (int r = 0; r < 4; r++) {
            uint32_t u[8], x2[8];
#pragma unroll
            for (int b = 0; b < 8; b++) u[b] = a[r * 8 + b] ^ a[((r + 1) & 3) * 8 + b];
            xtime8(u, x2);
#pragma unroll
            for (int b = 0; b < 8; b++) s[(c * 4 + r) * 8 + b] = a[r * 8 + b] ^ T[b] ^ x2[b] ^ c_rk[(c * 4 + r) * 8 + b];
        }
    }
}

// Inverse round (FIPS-197 §5.3 InvCipher order): InvShiftRows (renaming),
// InvSubBytes (tools/kg_inv_sbox_bp.cuh), AddRoundKey, InvMixColumns as
// MixColumns after the 04-multiple pre-step (a0 ^= 04(a0^a2), a2 likewise,
// a1 ^= 04(a1^a3), a3 likewise).
// Pin 8 values at this point of the (volatile-ordered) schedule: S-boxes
// bracketed by pins run one after another, which bounds the live registers
// (ptxas otherwise interleaves several S-boxes and spills).
__device__ __forceinline__ void pin8(uint32_t *x) {
    asm volatile("" : "+r"(x[0]), "+r"(x[1]), "+r"(x[2]), "+r"(x[3]), "+r"(x[4]), "+r"(x[5]), "+r"(x[6]), "+r"(x[7]));
}

__device__ __forceinline__ void bs_inv_round(uint32_t *s) {
    // InvSubBytes commutes with InvShiftRows: S-boxes in place on s first
#pragma unroll
    for (int byte = 0; byte < 16; byte++) {
        pin8(s + 8 * byte);
        bs_inv_sbox_bp(s + 8 * byte);
        pin8(s + 8 * byte);
    }
    uint32_t t[128];
#pragma unroll
    for (int c = 0; c < 4; c++)
#pragma unroll
        for (int r = 0; r < 4; r++)
#pragma unroll
            for (int b = 0; b < 8; b++)
                t[(c * 4 + r) * 8 + b] = s[(((c - r + 4) & 3) * 4 + r) * 8 + b] ^ c_rk[(c * 4 + r) * 8 + b];
    // InvMixColumns = MixColumns(e) with e_r = a_r ^ (r even ? U : V),
    // U = 04(a0^a2), V = 04(a1^a3).  The e sum equals the a sum T, and
    // e_r ^ e_{r+1} = a_r ^ a_{r+1} ^ U ^ V, so
    //   out_r = a_r ^ 02(a_r ^ a_{r+1}) ^ T ^ 02(U ^ V) ^ (r even ? U : V).
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

// one thread: a bitsliced inverse round on 32 blocks in[32][16] -> out[32][16]
__global__ void k_check_inv(const uint8_t *in, uint8_t *out) {
    if (threadIdx.x != 0) return;
    uint32_t s[128];
    for (int i = 0; i < 128; i++) s[i] = 0;
    for (int j = 0; j < 32; j++)
        for (int k = 0; k < 16; k++)  // byte k = row k%4, column k/4 (FIPS-197 §3.4)
            for (int b = 0; b < 8; b++) s[((k >> 2) * 4 + (k & 3)) * 8 + b] |= (uint32_t)((in[16 * j + k] >> b) & 1) << j;
    bs_inv_round(s);
    for (int j = 0; j < 32; j++)
        for (int k = 0; k < 16; k++) {
            int v = 0;
            for (int b = 0; b < 8; b++) v |= ((s[((k >> 2) * 4 + (k & 3)) * 8 + b] >> j) & 1) << b;
            out[16 * j + k] = (uint8_t)v;
        }
}

// NBS: bitsliced warps of warpgroup 3 (0..4); TT3: WG3's other warps run
// T-table rounds (else they exit at once)
template <int NTT_WG, int NBS, int SLEEP_SBOX, int SLEEP_ROUND, bool TT3 = false, bool INV = false>
__global__ void __launch_bounds__(512, 1) k_hybrid(unsigned long long ns, unsigned long long *cnt, uint32_t *sink) {
    extern __shared__ __align__(16) char smc[];
    for (int i = threadIdx.x; i < 32768; i += blockDim.x) reinterpret_cast<uint32_t *>(smc)[i] = i * 2654435761u;
    __syncthreads();
    const int wg = threadIdx.x >> 7;
    const int wiw = (threadIdx.x >> 5) & 3;  // warp in warpgroup
    const bool bs_role = NBS > 0 && wg == 3 && wiw < NBS;
    const bool tt_role = wg < NTT_WG || (TT3 && wg == 3 && !bs_role);
    unsigned long long g0, c0 = clock64();
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
    unsigned long long rounds = 0;
    if (NBS > 0) {
        if (wg == 3) asm volatile("setmaxnreg.inc.sync.aligned.u32 232;\n" ::);
        else asm volatile("setmaxnreg.dec.sync.aligned.u32 88;\n" ::);
    }
    if (tt_role) {
        const uint32_t l4 = (threadIdx.x & 31) * 4;
        const uint32_t lb = l4 | ((128u + l4) << 8);
        uint32_t a0 = threadIdx.x, a1 = threadIdx.x * 3, a2 = threadIdx.x * 5, a3 = threadIdx.x * 7;
        uint32_t b0 = threadIdx.x * 11, b1 = threadIdx.x * 13, b2 = threadIdx.x * 17, b3 = threadIdx.x * 19;
        const uint32_t k0 = 0x9e3779b9u;
#define TL(I, x) (*reinterpret_cast<const uint32_t *>(smc + (I >> 1) * 65536 + __byte_perm(x, lb, 0x7700u | (I << 4) | (4 + (I & 1)))))
        for (;;) {
#pragma unroll 1
            for (int it = 0; it < 64; it++) {
                uint32_t t0 = TL(0, a0) ^ TL(1, a1) ^ TL(2, a2) ^ TL(3, a3) ^ k0;
                uint32_t t1 = TL(0, a1) ^ TL(1, a2) ^ TL(2, a3) ^ TL(3, a0) ^ (k0 + 1);
                uint32_t t2 = TL(0, a2) ^ TL(1, a3) ^ TL(2, a0) ^ TL(3, a1) ^ (k0 + 2);
                uint32_t t3 = TL(0, a3) ^ TL(1, a0) ^ TL(2, a1) ^ TL(3, a2) ^ (k0 + 3);
                uint32_t u0 = TL(0, b0) ^ TL(1, b1) ^ TL(2, b2) ^ TL(3, b3) ^ k0;
                uint32_t u1 = TL(0, b1) ^ TL(1, b2) ^ TL(2, b3) ^ TL(3, b0) ^ (k0 + 1);
                uint32_t u2 = TL(0, b2) ^ TL(1, b3) ^ TL(2, b0) ^ TL(3, b1) ^ (k0 + 2);
                uint32_t u3 = TL(0, b3) ^ TL(1, b0) ^ TL(2, b1) ^ TL(3, b2) ^ (k0 + 3);
                a0 = t0; a1 = t1; a2 = t2; a3 = t3;
                b0 = u0; b1 = u1; b2 = u2; b3 = u3;
            }
            rounds += 64 * 2 * 32;  // block-rounds per warp (2 blocks per lane)
            unsigned long long g;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
            if (g - g0 > ns) break;
        }
#undef TL
        if ((a0 ^ a1 ^ a2 ^ a3 ^ b0 ^ b1 ^ b2 ^ b3) == 0xdeadbeef) sink[0] = 1;
    } else if (bs_role) {
        uint32_t s[128];
#pragma unroll
        for (int i = 0; i < 128; i++) s[i] = (threadIdx.x + 1) * (i + 7) * 2654435761u;
#pragma unroll 1
        for (;;) {
            if (INV) bs_inv_round(s);
            else bs_round<SLEEP_SBOX>(s);
            if (SLEEP_ROUND > 0) __nanosleep(SLEEP_ROUND);
            rounds += 32 * 32;  // 32 blocks per thread
            unsigned long long g;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
            if (g - g0 > ns) break;
        }
        uint32_t acc = 0;
#pragma unroll
        for (int i = 0; i < 128; i++) acc ^= s[i];
        if (acc == 0x12345678u) sink[0] = acc;
    }
    // every warp waits for the others, so the cycle count is the full interval
    __syncthreads();
    const unsigned long long c1 = clock64();
    if ((threadIdx.x & 31) == 0 && (tt_role || bs_role)) atomicAdd(&cnt[bs_role ? 1 : 0], rounds);
    if (threadIdx.x == 0) atomicMax(&cnt[2], c1 - c0);
}

template <int NTT_WG, int NBS, int SLEEP_SBOX, int SLEEP_ROUND, bool TT3 = false, bool INV = false>
static void run(int sms, const char *name) {
    unsigned long long *cnt;
    uint32_t *sink;
    cudaMalloc(&cnt, 32);
    cudaMalloc(&sink, 4);
    auto k = k_hybrid<NTT_WG, NBS, SLEEP_SBOX, SLEEP_ROUND, TT3, INV>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, k);
    for (int rep = 0; rep < 2; rep++) {
        cudaMemset(cnt, 0, 32);
        k<<<sms, 512, 131072>>>(5000000ull, cnt, sink);  // 5 ms
        cudaDeviceSynchronize();
    }
    unsigned long long h[4];
    cudaMemcpy(h, cnt, 32, cudaMemcpyDeviceToHost);
    const double clk = (double)h[2];
    printf("{\"test\": \"hybrid_throttle\", \"arm\": \"%s%s\", \"ttable_warps\": %d, \"bitsliced_warps\": %d, "
           "\"sleep_ns_per_sbox\": %d, \"sleep_ns_per_round\": %d, \"regs\": %d, \"local_bytes\": %zu, "
           "\"ttable_block_rounds_per_clk_sm\": %.4f, \"bitsliced_block_rounds_per_clk_sm\": %.4f, \"total\": %.4f, "
           "\"cycles\": %.0f}\n",
           name, INV ? "_inverse" : "", 4 * NTT_WG + (TT3 ? 4 - NBS : 0), NBS, SLEEP_SBOX, SLEEP_ROUND, fa.numRegs, (size_t)fa.localSizeBytes, h[0] / clk / sms,
           h[1] / clk / sms, (h[0] + h[1]) / clk / sms, clk);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("{\"error\": \"%s\"}\n", cudaGetErrorString(e));
    fflush(stdout);
    cudaFree(cnt);
    cudaFree(sink);
}

// host byte-oriented reference of one inverse round (for the device check)
static uint8_t gmul(uint8_t a, uint8_t b) {
    uint8_t p = 0;
    for (int i = 0; i < 8; i++) {
        if (b & 1) p ^= a;
        const uint8_t hi = a & 0x80;
        a <<= 1;
        if (hi) a ^= 0x1b;
        b >>= 1;
    }
    return p;
}

static bool check_inverse_round(const uint32_t *rk) {
    uint8_t sbox[256], isb[256];
    for (int x = 0; x < 256; x++) {
        uint8_t inv = 0;
        for (int y = 1; y < 256 && x; y++)
            if (gmul((uint8_t)x, (uint8_t)y) == 1) inv = (uint8_t)y;
        uint8_t b = inv, r = inv;
        for (int i = 0; i < 4; i++) {
            r = (uint8_t)((r << 1) | (r >> 7));
            b ^= r;
        }
        sbox[x] = b ^ 0x63;
    }
    for (int x = 0; x < 256; x++) isb[sbox[x]] = (uint8_t)x;
    uint8_t in[512], out[512], exp[512], key[16];
    for (int i = 0; i < 512; i++) in[i] = (uint8_t)(i * 131 + 7 + (i >> 4) * 29);
    for (int k = 0; k < 16; k++) {
        key[k] = 0;
        for (int b = 0; b < 8; b++) key[k] |= (uint8_t)((rk[k * 8 + b] & 1) << b);
    }
    for (int j = 0; j < 32; j++) {
        const uint8_t *o = in + 16 * j;
        uint8_t t[16];
        for (int c = 0; c < 4; c++)
            for (int r = 0; r < 4; r++) t[r + 4 * c] = isb[o[r + 4 * ((c - r + 4) & 3)]] ^ key[r + 4 * c];
        for (int c = 0; c < 4; c++)
            for (int r = 0; r < 4; r++)
                exp[16 * j + r + 4 * c] = gmul(t[r + 4 * c], 14) ^ gmul(t[(r + 1) % 4 + 4 * c], 11) ^
                                          gmul(t[(r + 2) % 4 + 4 * c], 13) ^ gmul(t[(r + 3) % 4 + 4 * c], 9);
    }
    uint8_t *d_in, *d_out;
    cudaMalloc(&d_in, 512);
    cudaMalloc(&d_out, 512);
    cudaMemcpy(d_in, in, 512, cudaMemcpyHostToDevice);
    k_check_inv<<<1, 32>>>(d_in, d_out);
    cudaMemcpy(out, d_out, 512, cudaMemcpyDeviceToHost);
    cudaFree(d_in);
    cudaFree(d_out);
    int bad = 0;
    for (int i = 0; i < 512; i++) bad += out[i] != exp[i];
    printf("{\"check\": \"bitsliced_inverse_round\", \"byte_mismatches\": %d}\n", bad);
    return bad == 0;
}

int main() {
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    uint32_t rk[128];
    for (int i = 0; i < 128; i++) rk[i] = (i * 2654435761u) & 0x10 ? 0xffffffffu : 0u;
    cudaMemcpyToSymbol(c_rk, rk, sizeof rk);
    const int sms = p.multiProcessorCount;
    check_inverse_round(rk);
    if (getenv("HYB_INV_ONLY")) {
        run<4, 0, 0, 0>(sms, "ttable_16w");
        run<3, 2, 0, 0, true, true>(sms, "hybrid_14tt_2bs");
        run<3, 3, 0, 0, true, true>(sms, "hybrid_13tt_3bs");
        run<3, 1, 0, 0, true, true>(sms, "hybrid_15tt_1bs");
        run<3, 2, 0, 0, false, true>(sms, "hybrid_2bs");
        return 0;
    }
    run<4, 0, 0, 0>(sms, "ttable_16w");
    run<3, 0, 0, 0>(sms, "ttable_12w");
    run<0, 4, 0, 0>(sms, "bitsliced_4w_alone");
    run<3, 4, 0, 0>(sms, "hybrid_free");
    run<3, 4, 32, 0>(sms, "hybrid_sleep_sbox");
    run<3, 4, 64, 0>(sms, "hybrid_sleep_sbox");
    run<3, 4, 128, 0>(sms, "hybrid_sleep_sbox");
    run<3, 4, 256, 0>(sms, "hybrid_sleep_sbox");
    run<3, 4, 512, 0>(sms, "hybrid_sleep_sbox");
    run<3, 4, 0, 1000>(sms, "hybrid_sleep_round");
    run<3, 4, 0, 2000>(sms, "hybrid_sleep_round");
    run<3, 4, 0, 4000>(sms, "hybrid_sleep_round");
    run<3, 2, 0, 0>(sms, "hybrid_2bs");
    run<3, 1, 0, 0>(sms, "hybrid_1bs");
    run<3, 2, 128, 0>(sms, "hybrid_2bs_sleep");
    run<3, 3, 0, 0>(sms, "hybrid_3bs");
    run<3, 2, 0, 0, true>(sms, "hybrid_14tt_2bs");
    run<3, 1, 0, 0, true>(sms, "hybrid_15tt_1bs");
    run<3, 3, 0, 0, true>(sms, "hybrid_13tt_3bs");
    run<3, 2, 64, 0, true>(sms, "hybrid_14tt_2bs_sleep");
    run<3, 2, 0, 0, true, true>(sms, "hybrid_14tt_2bs");
    run<3, 3, 0, 0, true, true>(sms, "hybrid_13tt_3bs");
    run<3, 1, 0, 0, true, true>(sms, "hybrid_15tt_1bs");
    run<3, 2, 0, 0, false, true>(sms, "hybrid_2bs");
    return 0;
}
