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

// NBS: bitsliced warps of warpgroup 3 (0..4); TT3: WG3's other warps run
// T-table rounds (else they exit at once)
template <int NTT_WG, int NBS, int SLEEP_SBOX, int SLEEP_ROUND, bool TT3 = false>
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
        for (;;) {
            bs_round<SLEEP_SBOX>(s);
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

template <int NTT_WG, int NBS, int SLEEP_SBOX, int SLEEP_ROUND, bool TT3 = false>
static void run(int sms, const char *name) {
    unsigned long long *cnt;
    uint32_t *sink;
    cudaMalloc(&cnt, 32);
    cudaMalloc(&sink, 4);
    auto k = k_hybrid<NTT_WG, NBS, SLEEP_SBOX, SLEEP_ROUND, TT3>;
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
    printf("{\"test\": \"hybrid_throttle\", \"arm\": \"%s\", \"ttable_warps\": %d, \"bitsliced_warps\": %d, "
           "\"sleep_ns_per_sbox\": %d, \"sleep_ns_per_round\": %d, \"regs\": %d, \"local_bytes\": %zu, "
           "\"ttable_block_rounds_per_clk_sm\": %.4f, \"bitsliced_block_rounds_per_clk_sm\": %.4f, \"total\": %.4f, "
           "\"cycles\": %.0f}\n",
           name, 4 * NTT_WG + (TT3 ? 4 - NBS : 0), NBS, SLEEP_SBOX, SLEEP_ROUND, fa.numRegs, (size_t)fa.localSizeBytes, h[0] / clk / sms,
           h[1] / clk / sms, (h[0] + h[1]) / clk / sms, clk);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("{\"error\": \"%s\"}\n", cudaGetErrorString(e));
    fflush(stdout);
    cudaFree(cnt);
    cudaFree(sink);
}

int main() {
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    uint32_t rk[128];
    for (int i = 0; i < 128; i++) rk[i] = (i * 2654435761u) & 0x10 ? 0xffffffffu : 0u;
    cudaMemcpyToSymbol(c_rk, rk, sizeof rk);
    const int sms = p.multiProcessorCount;
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
    return 0;
}
