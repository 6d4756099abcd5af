// pipes_ldpath.cu -- which L1TEX pipe do coalesced 16/32-byte global loads use?
// ld.global (LDG), ld.global.nc (__ldg), ld.global.nc.L1::no_allocate, and
// tex1Dfetch<uint4>: ncu's l1tex__data_pipe_lsu_wavefronts vs
// l1tex__data_pipe_tex_wavefronts tell whether a load path would compete with
// the shared-memory lookups (LSU data pipe) of the AES kernels.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

template <int V>
__global__ void k_load(const uint4 *__restrict__ p, cudaTextureObject_t tex, size_t n, uint4 *sink) {
    uint4 acc = make_uint4(0, 0, 0, 0);
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        uint4 v;
        if (V == 0) v = p[i];
        else if (V == 1) v = __ldg(p + i);
        else if (V == 2)
            asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p + i));
        else v = tex1Dfetch<uint4>(tex, (int)i);
        acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
    }
    if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345u) sink[0] = acc;
}

int main() {
    const size_t n = (256ull << 20) / 16;  // 256 MiB of uint4 (2^24 elements: within the 1D linear texture limit)
    uint4 *p, *sink;
    cudaMalloc(&p, n * 16);
    cudaMalloc(&sink, 16);
    cudaMemset(p, 1, n * 16);
    cudaResourceDesc rd = {};
    rd.resType = cudaResourceTypeLinear;
    rd.res.linear.devPtr = p;
    rd.res.linear.desc = cudaCreateChannelDesc<uint4>();
    rd.res.linear.sizeInBytes = n * 16;
    cudaTextureDesc td = {};
    td.readMode = cudaReadModeElementType;
    cudaTextureObject_t tex = 0;
    cudaError_t e = cudaCreateTextureObject(&tex, &rd, &td, nullptr);
    if (e != cudaSuccess) printf("{\"error\": \"tex: %s\"}\n", cudaGetErrorString(e));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const char *names[] = {"ld.global", "ld.global.nc", "ld.global.nc.L1::no_allocate", "tex1Dfetch"};
    for (int v = 0; v < 4; v++) {
        for (int rep = 0; rep < 2; rep++) {
            cudaEventRecord(a);
            if (v == 0) k_load<0><<<148 * 4, 512>>>(p, tex, n, sink);
            if (v == 1) k_load<1><<<148 * 4, 512>>>(p, tex, n, sink);
            if (v == 2) k_load<2><<<148 * 4, 512>>>(p, tex, n, sink);
            if (v == 3) k_load<3><<<148 * 4, 512>>>(p, tex, n, sink);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
        }
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("{\"test\": \"load_path\", \"path\": \"%s\", \"ms\": %.3f, \"gbs\": %.1f}\n", names[v], ms,
               n * 16 / (ms * 1e-3) / 1e9);
    }
    e = cudaGetLastError();
    if (e != cudaSuccess) printf("{\"error\": \"%s\"}\n", cudaGetErrorString(e));
    return 0;
}
