// bitslice_bench.cu -- throughput of one bitsliced AES encryption round
// (SubBytes via the generated tower-field circuit + ShiftRows (register
// renaming) + MixColumns + AddRoundKey) on 32 blocks per thread, in
// block-rounds per clock per SM, to compare with the T-table round of
// tools/pipes.cu (the north star's "T-table ... or a bitsliced LOP3 variant,
// whichever is faster").  No I/O, no transposes (those only add cost).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "kg_sbox_bs.cuh"

// state: s[(c*4 + r)*8 + b] = bit b of byte (row r, column c) of 32 blocks
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

__device__ __forceinline__ void bs_round(uint32_t *s, const uint32_t *rk /* 128 masks */) {
#pragma unroll
    for (int byte = 0; byte < 16; byte++) bs_sbox(s + 8 * byte);
    uint32_t t[128];
    // ShiftRows: byte (r, c) <- (r, c + r)
#pragma unroll
    for (int c = 0; c < 4; c++)
#pragma unroll
        for (int r = 0; r < 4; r++)
#pragma unroll
            for (int b = 0; b < 8; b++) t[(c * 4 + r) * 8 + b] = s[(((c + r) & 3) * 4 + r) * 8 + b];
    // MixColumns + AddRoundKey: out_r = a_r ^ T ^ 2(a_r ^ a_{r+1}) ^ k
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
            for (int b = 0; b < 8; b++) s[(c * 4 + r) * 8 + b] = a[r * 8 + b] ^ T[b] ^ x2[b] ^ rk[(c * 4 + r) * 8 + b];
        }
    }
}

__global__ void __launch_bounds__(128, 1) k_bs(uint32_t *sink, unsigned long long *cyc, int iters) {
    __shared__ uint32_t rk[128];
    if (threadIdx.x < 128) rk[threadIdx.x] = (threadIdx.x * 2654435761u) & 1 ? 0xffffffffu : 0u;
    __syncthreads();
    uint32_t s[128];
#pragma unroll
    for (int i = 0; i < 128; i++) s[i] = (threadIdx.x + 1) * (i + 7) * 2654435761u;
    uint32_t k[128];
#pragma unroll
    for (int i = 0; i < 128; i++) k[i] = rk[i];
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; it++) bs_round(s, k);
    __syncthreads();
    unsigned long long t1 = clock64();
    uint32_t acc = 0;
#pragma unroll
    for (int i = 0; i < 128; i++) acc ^= s[i];
    if (acc == 0x12345678u) sink[0] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    const int sms = p.multiProcessorCount;
    uint32_t *sink;
    unsigned long long *cyc;
    cudaMalloc(&sink, 4);
    cudaMalloc(&cyc, 8 * sms * 16);
    for (int wps : {4, 8, 12, 16}) {  // warps per SM: blocks of 128 threads, wps/4 blocks per SM
        const int blocks_per_sm = wps / 4;
        const int iters = 200;
        k_bs<<<sms * blocks_per_sm, 128>>>(sink, cyc, iters);
        cudaDeviceSynchronize();
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        k_bs<<<sms * blocks_per_sm, 128>>>(sink, cyc, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        unsigned long long h[4096];
        cudaMemcpy(h, cyc, 8 * sms * blocks_per_sm, cudaMemcpyDeviceToHost);
        unsigned long long mx = 0;
        for (int i = 0; i < sms * blocks_per_sm; i++) mx = h[i] > mx ? h[i] : mx;
        const double block_rounds_per_sm = (double)blocks_per_sm * 128 * 32 * iters;
        printf("{\"test\": \"bitsliced_round\", \"warps_per_sm\": %d, \"block_rounds_per_clk_sm\": %.3f}\n", wps,
               block_rounds_per_sm / mx);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("{\"error\": \"%s\"}\n", cudaGetErrorString(e));
    return 0;
}
