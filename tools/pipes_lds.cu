// pipes_lds.cu -- shared-memory load/store bytes per clock per SM by access
// width (LDS.32/.64/.128, STS.128), conflict-free, and LDG.256 from L2-resident
// data: is the LSU data pipe 128 B per wavefront for every width?  Kernel
// durations come from ncu / CUDA events; SM clock from clock64 over the same
// loop (printed per test).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

constexpr int kThreads = 1024;
constexpr int kIters = 2048;

template <int W>  // words per lane access: 1, 2, 4
__global__ void __launch_bounds__(kThreads, 1) k_lds(uint32_t *sink, unsigned long long *cyc) {
    extern __shared__ __align__(16) uint32_t sm[];
    for (int i = threadIdx.x; i < 16384; i += blockDim.x) sm[i] = i * 2654435761u;
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31;
    uint32_t acc[4] = {0, 0, 0, 0};
    uint32_t x = threadIdx.x;
    unsigned long long t0 = clock64();
    for (int it = 0; it < kIters; it++) {
#pragma unroll
        for (int c = 0; c < 8; c++) {
            // row r (dependent on the last value, so loads are not hoisted), lane-contiguous W words
            const uint32_t r = (x + c) & 63;
            const uint32_t *p = sm + r * (32 * W) + lane * W;
            if (W == 1) {
                x += p[0];
            } else if (W == 2) {
                const uint2 v = *reinterpret_cast<const uint2 *>(p);
                x += v.x ^ v.y;
            } else {
                const uint4 v = *reinterpret_cast<const uint4 *>(p);
                x += v.x ^ v.y ^ v.z ^ v.w;
            }
        }
    }
    __syncthreads();
    unsigned long long t1 = clock64();
    if (x == 0xdeadbeef) sink[0] = x + acc[0];
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// independent (not dependent-chained) LDS.128: 8 loads in flight per thread
template <int W>
__global__ void __launch_bounds__(kThreads, 1) k_lds_ilp(uint32_t *sink, unsigned long long *cyc) {
    extern __shared__ __align__(16) uint32_t sm[];
    for (int i = threadIdx.x; i < 16384; i += blockDim.x) sm[i] = i * 2654435761u;
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31;
    uint32_t x[8];
#pragma unroll
    for (int c = 0; c < 8; c++) x[c] = c;
    unsigned long long t0 = clock64();
    for (int it = 0; it < kIters; it++) {
#pragma unroll
        for (int c = 0; c < 8; c++) {
            const uint32_t r = (x[c] + c) & 63;
            const uint32_t *p = sm + r * (32 * W) + lane * W;
            if (W == 1) {
                x[c] += p[0];
            } else if (W == 2) {
                const uint2 v = *reinterpret_cast<const uint2 *>(p);
                x[c] += v.x ^ v.y;
            } else {
                const uint4 v = *reinterpret_cast<const uint4 *>(p);
                x[c] += v.x ^ v.y ^ v.z ^ v.w;
            }
        }
    }
    __syncthreads();
    unsigned long long t1 = clock64();
    uint32_t a = 0;
#pragma unroll
    for (int c = 0; c < 8; c++) a ^= x[c];
    if (a == 0xdeadbeef) sink[0] = a;
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

template <int W>
static void run(const char *name, void (*k)(uint32_t *, unsigned long long *), int sms, uint32_t *sink,
                unsigned long long *cyc) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k<<<sms, kThreads, 65536>>>(sink, cyc);
    cudaEventRecord(e0);
    k<<<sms, kThreads, 65536>>>(sink, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double c = median_cycles(cyc, sms);
    const double bytes = (double)kThreads * kIters * 8 * 4 * W;  // per SM
    printf("{\"test\": \"%s\", \"bytes_per_lane_access\": %d, \"bytes_per_clk_sm\": %.1f, \"ms\": %.3f, \"mhz\": %.0f}\n",
           name, 4 * W, bytes / c, ms, c / (ms * 1e3));
}

int main() {
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    const int sms = p.multiProcessorCount;
    uint32_t *sink;
    unsigned long long *cyc;
    cudaMalloc(&sink, 4);
    cudaMalloc(&cyc, sizeof(unsigned long long) * sms);
    run<1>("lds_dep", k_lds<1>, sms, sink, cyc);
    run<2>("lds_dep", k_lds<2>, sms, sink, cyc);
    run<4>("lds_dep", k_lds<4>, sms, sink, cyc);
    run<1>("lds_ilp", k_lds_ilp<1>, sms, sink, cyc);
    run<2>("lds_ilp", k_lds_ilp<2>, sms, sink, cyc);
    run<4>("lds_ilp", k_lds_ilp<4>, sms, sink, cyc);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("{\"error\": \"%s\"}\n", cudaGetErrorString(e));
    return 0;
}
