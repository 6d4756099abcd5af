// pipes.cu -- per-SM pipe-rate microbenchmarks: the roofline inputs for the
// T-table AES kernels.  One CTA of 1024 threads per SM,
// timed in SM cycles with clock64() inside each CTA, so the results are
// clock-independent (lane-ops per SM-cycle).
//
//   lds   : lane-private-bank LDS.32 (the T-table access pattern: lane l only
//           touches bank l), 8 independent chains per thread
//   prmt  : PRMT throughput, 8 independent chains
//   lop3  : 3-input LOP3 throughput, 8 independent chains
//   round : one full T-table AES round per iteration (16 PRMT + 16 LDS + 8 LOP3)
//
// Output: one JSON line per test {"test", "lane_ops_per_clk_sm", ...}.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

constexpr int kThreads = 1024;
constexpr int kIters = 4096;

__global__ void __launch_bounds__(kThreads, 1) k_lds(uint32_t *sink, unsigned long long *cyc) {
    extern __shared__ uint32_t sm[];
    const uint32_t lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 16384; i += blockDim.x) sm[i] = (i * 2654435761u) & 0x1ff;
    __syncthreads();
    uint32_t x[8];
#pragma unroll
    for (int c = 0; c < 8; c++) x[c] = c;
    unsigned long long t0 = clock64();
    for (int it = 0; it < kIters; it++) {
#pragma unroll
        for (int c = 0; c < 8; c++) x[c] = sm[((x[c] & 0x1ff) << 5) | lane];  // bank = lane
    }
    __syncthreads();
    unsigned long long t1 = clock64();
    uint32_t acc = 0;
#pragma unroll
    for (int c = 0; c < 8; c++) acc ^= x[c];
    if (acc == 0xdeadbeef) sink[0] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void __launch_bounds__(kThreads, 1) k_prmt(uint32_t *sink, unsigned long long *cyc, uint32_t seed) {
    uint32_t x[8];
#pragma unroll
    for (int c = 0; c < 8; c++) x[c] = seed + c + threadIdx.x;
    unsigned long long t0 = clock64();
    for (int it = 0; it < kIters; it++) {
#pragma unroll
        for (int c = 0; c < 8; c++) x[c] = __byte_perm(x[c], seed, 0x7415 + c);
    }
    __syncthreads();
    unsigned long long t1 = clock64();
    uint32_t acc = 0;
#pragma unroll
    for (int c = 0; c < 8; c++) acc ^= x[c];
    if (acc == 0xdeadbeef) sink[0] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void __launch_bounds__(kThreads, 1) k_lop3(uint32_t *sink, unsigned long long *cyc, uint32_t seed) {
    uint32_t x[8];
#pragma unroll
    for (int c = 0; c < 8; c++) x[c] = seed * (c + 1) + threadIdx.x;
    const uint32_t y = seed ^ 0x5a5a5a5a, z = seed + 77;
    unsigned long long t0 = clock64();
    for (int it = 0; it < kIters; it++) {
#pragma unroll
        for (int c = 0; c < 8; c++) {
            uint32_t r;
            asm volatile("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(r) : "r"(x[c]), "r"(y + c), "r"(z));
            x[c] = r;
        }
    }
    __syncthreads();
    unsigned long long t1 = clock64();
    uint32_t acc = 0;
#pragma unroll
    for (int c = 0; c < 8; c++) acc ^= x[c];
    if (acc == 0xdeadbeef) sink[0] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// One T-table round per iteration on one block per thread, same layout and
// instruction mix as the library kernels.
__global__ void __launch_bounds__(kThreads, 1) k_round(uint32_t *sink, unsigned long long *cyc, uint32_t k0) {
    extern __shared__ __align__(16) char smc[];
    for (int i = threadIdx.x; i < 32768; i += blockDim.x) reinterpret_cast<uint32_t *>(smc)[i] = i * 2654435761u;
    __syncthreads();
    const uint32_t l4 = (threadIdx.x & 31) * 4;
    const uint32_t lb = l4 | ((128u + l4) << 8);
    uint32_t s0 = threadIdx.x, s1 = threadIdx.x * 3, s2 = threadIdx.x * 5, s3 = threadIdx.x * 7;
#define TL(I, x) (*reinterpret_cast<const uint32_t *>(smc + (I >> 1) * 65536 + __byte_perm(x, lb, 0x7700u | (I << 4) | (4 + (I & 1)))))
    unsigned long long t0 = clock64();
    for (int it = 0; it < kIters / 4; it++) {
        uint32_t t0_ = TL(0, s0) ^ TL(1, s1) ^ TL(2, s2) ^ TL(3, s3) ^ k0;
        uint32_t t1_ = TL(0, s1) ^ TL(1, s2) ^ TL(2, s3) ^ TL(3, s0) ^ (k0 + 1);
        uint32_t t2_ = TL(0, s2) ^ TL(1, s3) ^ TL(2, s0) ^ TL(3, s1) ^ (k0 + 2);
        uint32_t t3_ = TL(0, s3) ^ TL(1, s0) ^ TL(2, s1) ^ TL(3, s2) ^ (k0 + 3);
        s0 = t0_; s1 = t1_; s2 = t2_; s3 = t3_;
    }
#undef TL
    __syncthreads();
    unsigned long long t1 = clock64();
    if ((s0 ^ s1 ^ s2 ^ s3) == 0xdeadbeef) sink[0] = s0;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

static double median_cycles(unsigned long long *d, int n) {
    unsigned long long h[1024];
    cudaMemcpy(h, d, n * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    for (int i = 0; i < n; i++)
        for (int j = i + 1; j < n; j++)
            if (h[j] < h[i]) { unsigned long long t = h[i]; h[i] = h[j]; h[j] = t; }
    return (double)h[n / 2];
}

int main() {
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    const int sms = p.multiProcessorCount;
    uint32_t *sink;
    unsigned long long *cyc;
    cudaMalloc(&sink, 4);
    cudaMalloc(&cyc, sizeof(unsigned long long) * sms);
    cudaFuncSetAttribute(k_lds, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    cudaFuncSetAttribute(k_round, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
    const double lane_ops_8 = (double)kThreads * kIters * 8;
    for (int rep = 0; rep < 2; rep++) {
        k_lds<<<sms, kThreads, 65536>>>(sink, cyc);
        cudaDeviceSynchronize();
        double c = median_cycles(cyc, sms);
        if (rep) printf("{\"test\": \"lds_lane_private\", \"lane_ops_per_clk_sm\": %.2f, \"sms\": %d}\n", lane_ops_8 / c, sms);
        k_prmt<<<sms, kThreads>>>(sink, cyc, 12345);
        cudaDeviceSynchronize();
        c = median_cycles(cyc, sms);
        if (rep) printf("{\"test\": \"prmt\", \"lane_ops_per_clk_sm\": %.2f}\n", lane_ops_8 / c);
        k_lop3<<<sms, kThreads>>>(sink, cyc, 12345);
        cudaDeviceSynchronize();
        c = median_cycles(cyc, sms);
        if (rep) printf("{\"test\": \"lop3\", \"lane_ops_per_clk_sm\": %.2f}\n", lane_ops_8 / c);
        k_round<<<sms, kThreads, 131072>>>(sink, cyc, 777);
        cudaDeviceSynchronize();
        c = median_cycles(cyc, sms);
        const double rounds = (double)kThreads * (kIters / 4);
        if (rep)
            printf("{\"test\": \"aes_round_ttable\", \"block_rounds_per_clk_sm\": %.3f, \"lds_per_clk_sm\": %.2f}\n",
                   rounds / c, rounds * 16 / c);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        printf("{\"error\": \"%s\"}\n", cudaGetErrorString(e));
        return 1;
    }
    return 0;
}
