// copy_overlap.cu -- why do H2D and D2H chunks not overlap in the staging
// pipeline?  Reproduces the pipeline's stream/event structure with plain
// CUDA (no libkgpu) in several variants and prints the total time of a
// 256 MiB pinned->device->pinned pass for each.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <vector>

// occupies every SM (1 CTA of 1024 threads + 192 KB smem per SM) for ~`ns`
__global__ void spin_kernel(unsigned long long ns) {
    extern __shared__ char smem_dummy[];
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > ns) break;
    }
    if (threadIdx.x == 5000) smem_dummy[0] = 1;
}

__global__ void noop_kernel(uint4 *p, size_t n) {
    if (n == 0xFFFFFFFFFFFull) p[threadIdx.x] = make_uint4(0, 0, 0, 0);
}

__global__ void touch(uint4 *p, size_t n) {
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    for (; i < n; i += (size_t)gridDim.x * blockDim.x) {
        uint4 v = p[i];
        v.x ^= 1;
        p[i] = v;
    }
}

static int g_kernel_kind = 0;  // 0 touch<<<148,1024>>>, 1 noop<<<148,1024,smem>>>, 2 noop<<<1,32>>>
static float run(const char *name, uint8_t *hin, uint8_t *hout, uint8_t **stage, int slots, size_t total, size_t chunk,
                 bool with_kernel, bool events, cudaStream_t sh, cudaStream_t sk, cudaStream_t sd, int smem) {
    std::vector<cudaEvent_t> loaded(slots), done(slots), freed(slots);
    for (int i = 0; i < slots; i++) {
        cudaEventCreateWithFlags(&loaded[i], cudaEventDisableTiming);
        cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming);
        cudaEventCreateWithFlags(&freed[i], cudaEventDisableTiming);
    }
    cudaEvent_t t0, t1;
    cudaEventCreate(&t0);
    cudaEventCreate(&t1);
    float best = 1e9f;
    for (int rep = 0; rep < 4; rep++) {
        cudaDeviceSynchronize();
        cudaEventRecord(t0, sh);
        cudaStreamWaitEvent(sd, t0, 0);
        cudaStreamWaitEvent(sk, t0, 0);
        size_t nch = (total + chunk - 1) / chunk;
        for (size_t i = 0; i < nch; i++) {
            int s = (int)(i % slots);
            size_t off = i * chunk, nb = (total - off < chunk) ? total - off : chunk;
            if (events) cudaStreamWaitEvent(sh, freed[s], 0);
            cudaMemcpyAsync(stage[s], hin + off, nb, cudaMemcpyHostToDevice, sh);
            if (events) cudaEventRecord(loaded[s], sh);
            if (with_kernel) {
                if (events) cudaStreamWaitEvent(sk, loaded[s], 0);
                if (g_kernel_kind == 0) touch<<<148, 1024, smem, sk>>>((uint4 *)stage[s], nb / 16);
                else if (g_kernel_kind == 1) noop_kernel<<<148, 1024, smem, sk>>>((uint4 *)stage[s], nb / 16);
                else noop_kernel<<<1, 32, 0, sk>>>((uint4 *)stage[s], nb / 16);
                if (events) cudaEventRecord(done[s], sk);
                if (events) cudaStreamWaitEvent(sd, done[s], 0);
            } else if (events) {
                cudaStreamWaitEvent(sd, loaded[s], 0);
            }
            cudaMemcpyAsync(hout + off, stage[s], nb, cudaMemcpyDeviceToHost, sd);
            if (events) cudaEventRecord(freed[s], sd);
        }
        cudaEventRecord(t1, sd);
        cudaEventSynchronize(t1);
        float ms;
        cudaEventElapsedTime(&ms, t0, t1);
        if (ms < best) best = ms;
    }
    printf("{\"variant\": \"%s\", \"chunk_mib\": %zu, \"smem\": %d, \"ms\": %.3f, \"gbs\": %.2f}\n", name, chunk >> 20, smem,
           best, total / (best * 1e-3) / 1e9);
    return best;
}

__global__ void zc_copy(const uint4 *__restrict__ src, uint4 *__restrict__ dst, size_t n) {
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
#pragma unroll 4
    for (; i < n; i += stride) dst[i] = src[i];
}

static void zc(const char *name, const uint8_t *src, uint8_t *dst, size_t total, int blocks, int threads) {
    cudaEvent_t t0, t1;
    cudaEventCreate(&t0);
    cudaEventCreate(&t1);
    float best = 1e9f;
    for (int rep = 0; rep < 4; rep++) {
        cudaEventRecord(t0);
        zc_copy<<<blocks, threads>>>((const uint4 *)src, (uint4 *)dst, total / 16);
        cudaEventRecord(t1);
        cudaEventSynchronize(t1);
        float ms;
        cudaEventElapsedTime(&ms, t0, t1);
        if (ms < best) best = ms;
    }
    printf("{\"variant\": \"%s\", \"blocks\": %d, \"threads\": %d, \"ms\": %.3f, \"gbs\": %.2f}\n", name, blocks, threads,
           best, total / (best * 1e-3) / 1e9);
}

// hybrid pipelines: one direction by copy engine, the other by the kernel itself
static void hybrid(const char *name, bool kernel_writes_host, uint8_t *hin, uint8_t *hout, uint8_t **stage, int slots,
                   size_t total, size_t chunk, cudaStream_t sh, cudaStream_t sk) {
    std::vector<cudaEvent_t> loaded(slots), freed(slots);
    for (int i = 0; i < slots; i++) {
        cudaEventCreateWithFlags(&loaded[i], cudaEventDisableTiming);
        cudaEventCreateWithFlags(&freed[i], cudaEventDisableTiming);
    }
    cudaEvent_t t0, t1;
    cudaEventCreate(&t0);
    cudaEventCreate(&t1);
    float best = 1e9f;
    for (int rep = 0; rep < 4; rep++) {
        cudaDeviceSynchronize();
        cudaEventRecord(t0, sh);
        cudaStreamWaitEvent(sk, t0, 0);
        size_t nch = (total + chunk - 1) / chunk;
        for (size_t i = 0; i < nch; i++) {
            int s = (int)(i % slots);
            size_t off = i * chunk, nb = (total - off < chunk) ? total - off : chunk;
            if (kernel_writes_host) {
                cudaStreamWaitEvent(sh, freed[s], 0);
                cudaMemcpyAsync(stage[s], hin + off, nb, cudaMemcpyHostToDevice, sh);
                cudaEventRecord(loaded[s], sh);
                cudaStreamWaitEvent(sk, loaded[s], 0);
                zc_copy<<<148, 1024, 0, sk>>>((const uint4 *)stage[s], (uint4 *)(hout + off), nb / 16);
                cudaEventRecord(freed[s], sk);
            } else {
                cudaStreamWaitEvent(sk, freed[s], 0);
                zc_copy<<<148, 1024, 0, sk>>>((const uint4 *)(hin + off), (uint4 *)stage[s], nb / 16);
                cudaEventRecord(loaded[s], sk);
                cudaStreamWaitEvent(sh, loaded[s], 0);
                cudaMemcpyAsync(hout + off, stage[s], nb, cudaMemcpyDeviceToHost, sh);
                cudaEventRecord(freed[s], sh);
            }
        }
        cudaEventRecord(t1, kernel_writes_host ? sk : sh);
        cudaEventSynchronize(t1);
        float ms;
        cudaEventElapsedTime(&ms, t0, t1);
        if (ms < best) best = ms;
    }
    printf("{\"variant\": \"%s\", \"chunk_mib\": %zu, \"ms\": %.3f, \"gbs\": %.2f}\n", name, chunk >> 20, best,
           total / (best * 1e-3) / 1e9);
}

int main() {
    const size_t total = 256ull << 20;
    uint8_t *hin, *hout;
    cudaHostAlloc(&hin, total, 0);
    cudaHostAlloc(&hout, total, 0);
    uint8_t *stage[8];
    for (int i = 0; i < 8; i++) cudaMalloc(&stage[i], 64ull << 20);
    cudaStream_t sh, sk, sd;
    cudaStreamCreateWithFlags(&sh, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&sk, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&sd, cudaStreamNonBlocking);
    cudaFuncSetAttribute(touch, cudaFuncAttributeMaxDynamicSharedMemorySize, 196480);
    uint8_t *dbuf, *dbuf2;
    cudaMalloc(&dbuf, total);
    cudaMalloc(&dbuf2, total);
    for (int b : {148, 296, 1184}) {
        zc("zc_read_pinned_to_hbm", hin, dbuf, total, b, 1024);
        zc("zc_write_hbm_to_pinned", dbuf, hout, total, b, 1024);
        zc("zc_pinned_to_pinned", hin, hout, total, b, 1024);
    }
    cudaFuncSetAttribute(noop_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 196480);
    cudaFuncSetAttribute(spin_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 196480);
    {
        // copies (no kernels) while a GPU-filling kernel spins on another stream
        cudaStream_t sx;
        cudaStreamCreateWithFlags(&sx, cudaStreamNonBlocking);
        cudaEvent_t a0, a1;
        cudaEventCreate(&a0);
        cudaEventCreate(&a1);
        for (int busy = 0; busy < 2; busy++) {
            cudaDeviceSynchronize();
            if (busy) spin_kernel<<<148, 1024, 196480, sx>>>(20000000ull);  // 20 ms
            cudaEventRecord(a0, sh);
            cudaMemcpyAsync(stage[0], hin, 64ull << 20, cudaMemcpyHostToDevice, sh);
            cudaEventRecord(a1, sh);
            cudaEventSynchronize(a1);
            float ms;
            cudaEventElapsedTime(&ms, a0, a1);
            printf("{\"variant\": \"h2d_64MiB_%s\", \"ms\": %.3f, \"gbs\": %.2f}\n", busy ? "while_gpu_full" : "idle",
                   ms, (64 << 20) / (ms * 1e-3) / 1e9);
            cudaEventRecord(a0, sd);
            cudaMemcpyAsync(hout, stage[1], 64ull << 20, cudaMemcpyDeviceToHost, sd);
            cudaEventRecord(a1, sd);
            cudaEventSynchronize(a1);
            cudaEventElapsedTime(&ms, a0, a1);
            printf("{\"variant\": \"d2h_64MiB_%s\", \"ms\": %.3f, \"gbs\": %.2f}\n", busy ? "while_gpu_full" : "idle",
                   ms, (64 << 20) / (ms * 1e-3) / 1e9);
            cudaDeviceSynchronize();
        }
    }
    for (size_t c : {8ull << 20, 16ull << 20}) {
        run("copies_events", hin, hout, stage, 3, total, c, false, true, sh, sk, sd, 0);
        g_kernel_kind = 0;
        run("touch_kernel_events", hin, hout, stage, 3, total, c, true, true, sh, sk, sd, 0);
        g_kernel_kind = 1;
        run("noop148x1024_kernel_events", hin, hout, stage, 3, total, c, true, true, sh, sk, sd, 0);
        run("noop148x1024_192KB_kernel_events", hin, hout, stage, 3, total, c, true, true, sh, sk, sd, 196480);
        g_kernel_kind = 2;
        run("noop1x32_kernel_events", hin, hout, stage, 3, total, c, true, true, sh, sk, sd, 0);
        g_kernel_kind = 0;
    }
    for (size_t c : {1ull << 20, 4ull << 20, 8ull << 20, 16ull << 20}) {
        hybrid("ce_h2d+kernel_writes_host", true, hin, hout, stage, 3, total, c, sh, sk);
        hybrid("kernel_reads_host+ce_d2h", false, hin, hout, stage, 3, total, c, sh, sk);
    }
    for (size_t c : {2ull << 20, 4ull << 20, 16ull << 20, 32ull << 20, 64ull << 20})
        run("copies_only_no_events(stage reuse unsafe)", hin, hout, stage, 3, total, c, false, false, sh, sk, sd, 0);
    for (size_t c : {1ull << 20, 8ull << 20}) {
        run("copies_only_no_events(stage reuse unsafe)", hin, hout, stage, 3, total, c, false, false, sh, sk, sd, 0);
        run("copies_events", hin, hout, stage, 3, total, c, false, true, sh, sk, sd, 0);
        run("copies_kernel_events", hin, hout, stage, 3, total, c, true, true, sh, sk, sd, 0);
        run("copies_kernel_events_192KBsmem", hin, hout, stage, 3, total, c, true, true, sh, sk, sd, 196480);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("{\"error\": \"%s\"}\n", cudaGetErrorString(e));
    return 0;
}
