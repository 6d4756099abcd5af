// pipe_variants.cu -- where does the staged pinned pipeline lose against the
// contended link rate?  256 MiB pinned -> HBM -> pinned in 16 MiB chunks with
// plenty of device slots (no slot-reuse waits), 5 variants of the compute
// step between a chunk's H2D and its D2H.  Reports total GB/s and when the
// H2D stream alone finished (GB/s of the H2D stream).
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <atomic>
#include <thread>
#include <vector>

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

// occupies every SM for ~ns (optionally with a large dynamic smem allocation)
__global__ void spin(unsigned long long ns) {
    extern __shared__ char smem_dummy[];
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    do {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    } while (t - t0 < ns);
    if (threadIdx.x == 5000) smem_dummy[0] = 1;
}

// persistent: processes chunk c once flag_in[c] == 1 (set by the H2D stream
// with a stream memory op), then sets flag_out[c] = 1 (device memory,
// release) for the D2H stream's wait-value.
__global__ void persistent(uint8_t *stage, size_t chunk, int nch, volatile uint32_t *flag_in, uint32_t *flag_out,
                           uint32_t *count) {
    for (int c = 0; c < nch; c++) {
        if (threadIdx.x == 0) {
            for (long spin = 0; flag_in[c] == 0 && spin < (1l << 25); spin++) __nanosleep(200);
            __threadfence();
        }
        __syncthreads();
        uint4 *p = (uint4 *)(stage + c * chunk);
        const size_t n = chunk / 16;
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
            uint4 v = p[i];
            v.x ^= 1;
            p[i] = v;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            if (atomicAdd(&count[c], 1) == gridDim.x - 1) {
                __threadfence();
                atomicExch(&flag_out[c], 1u);
            }
        }
    }
}

int main() {
    const size_t total = 256ull << 20, chunk = 16ull << 20;
    const int nch = (int)(total / chunk);
    uint8_t *hin, *hout, *dstage;
    cudaHostAlloc(&hin, total, 0);
    cudaHostAlloc(&hout, total, 0);
    cudaMalloc(&dstage, total);
    uint32_t *flags;
    cudaMalloc(&flags, 3 * 64 * sizeof(uint32_t));
    cudaStream_t sh, sk, sd;
    cudaStreamCreateWithFlags(&sh, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&sk, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&sd, cudaStreamNonBlocking);
    std::vector<cudaEvent_t> loaded(nch), done(nch);
    for (int i = 0; i < nch; i++) {
        cudaEventCreateWithFlags(&loaded[i], cudaEventDisableTiming);
        cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming);
    }
    cudaEvent_t t0, th, td;
    cudaEventCreate(&t0);
    cudaEventCreate(&th);
    cudaEventCreate(&td);
    const char *names[] = {"copies_no_deps", "events_no_kernel", "events_noop_kernel", "events_touch_kernel",
                           "memops_persistent_kernel", "events_spin30us_nosmem", "events_spin30us_smem196K",
                           "events_spin30us_smem196K_1cta", "events_spin10us_smem196K",
                           "lagged_d2h_spin30us", "lagged_d2h_touch", "lagged2_d2h_spin30us"};
    cudaFuncSetAttribute(spin, cudaFuncAttributeMaxDynamicSharedMemorySize, 196608);
    for (int v = 0; v < 12; v++) {
        float best = 1e9f, besth = 1e9f;
        for (int rep = 0; rep < 5; rep++) {
            cudaMemset(flags, 0, 3 * 64 * sizeof(uint32_t));
            cudaDeviceSynchronize();
            cudaEventRecord(t0, sh);
            cudaStreamWaitEvent(sk, t0, 0);
            cudaStreamWaitEvent(sd, t0, 0);
            if (v == 4)
                persistent<<<148, 1024, 0, sk>>>(dstage, chunk, nch, flags, flags + 64, flags + 128);
            if (v >= 9) {
                // D2H(i) additionally waits for H2D(i+lag): the D2H of a chunk starts together
                // with an H2D, never in the middle of one
                const int lag = v == 11 ? 2 : 1;
                for (int i = 0; i < nch + lag; i++) {
                    if (i < nch) {
                        cudaMemcpyAsync(dstage + i * chunk, hin + i * chunk, chunk, cudaMemcpyHostToDevice, sh);
                        cudaEventRecord(loaded[i], sh);
                        cudaStreamWaitEvent(sk, loaded[i], 0);
                        if (v == 10) touch<<<148, 1024, 0, sk>>>((uint4 *)(dstage + i * chunk), chunk / 16);
                        else spin<<<148, 512, 196608, sk>>>(30000);
                        cudaEventRecord(done[i], sk);
                    }
                    const int j = i - lag;
                    if (j >= 0) {
                        cudaStreamWaitEvent(sd, done[j], 0);
                        if (i < nch) cudaStreamWaitEvent(sd, loaded[i], 0);
                        cudaMemcpyAsync(hout + j * chunk, dstage + j * chunk, chunk, cudaMemcpyDeviceToHost, sd);
                    }
                }
            }
            for (int i = 0; i < nch && v < 9; i++) {
                uint8_t *st = dstage + i * chunk;
                cudaMemcpyAsync(st, hin + i * chunk, chunk, cudaMemcpyHostToDevice, sh);
                if (v == 4) {
                    cuStreamWriteValue32((CUstream)sh, (CUdeviceptr)(flags + i), 1, 0);
                    cuStreamWaitValue32((CUstream)sd, (CUdeviceptr)(flags + 64 + i), 1, CU_STREAM_WAIT_VALUE_GEQ);
                } else if (v >= 1) {
                    cudaEventRecord(loaded[i], sh);
                    if (v >= 2) {
                        cudaStreamWaitEvent(sk, loaded[i], 0);
                        if (v == 2) noop_kernel<<<1, 32, 0, sk>>>((uint4 *)st, chunk / 16);
                        else if (v == 3) touch<<<148, 1024, 0, sk>>>((uint4 *)st, chunk / 16);
                        else if (v == 5) spin<<<148, 512, 0, sk>>>(30000);
                        else if (v == 6) spin<<<148, 512, 196608, sk>>>(30000);
                        else if (v == 7) spin<<<1, 512, 196608, sk>>>(30000);
                        else spin<<<148, 512, 196608, sk>>>(10000);
                        cudaEventRecord(done[i], sk);
                        cudaStreamWaitEvent(sd, done[i], 0);
                    } else {
                        cudaStreamWaitEvent(sd, loaded[i], 0);
                    }
                }
                cudaMemcpyAsync(hout + i * chunk, st, chunk, cudaMemcpyDeviceToHost, sd);
            }
            cudaEventRecord(th, sh);
            cudaEventRecord(td, sd);
            cudaDeviceSynchronize();
            float ms, msh;
            cudaEventElapsedTime(&ms, t0, td);
            cudaEventElapsedTime(&msh, t0, th);
            if (ms < best) best = ms, besth = msh;
        }
        printf("{\"variant\": \"%s\", \"chunk_mib\": 16, \"ms\": %.3f, \"gbs\": %.2f, \"h2d_stream_gbs\": %.2f}\n",
               names[v], best, total / (best * 1e-3) / 1e9, total / (besth * 1e-3) / 1e9);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) printf("{\"error\": \"%s\"}\n", cudaGetErrorString(e));
    }
    // host-issued D2H: a second host thread waits for each chunk's kernel and only
    // then enqueues its D2H, so the D2H channel never holds a semaphore wait
    const int spins[] = {30000, 0, 5000, 10000, 20000, 30000, 50000, -1, -2};
    for (int kx = 0; kx < 9; kx++) {
        const int kk = spins[kx] >= 0 ? 0 : (spins[kx] == -1 ? 1 : 2);
        float best = 1e9f, besth = 1e9f;
        for (int rep = 0; rep < 5; rep++) {
            cudaDeviceSynchronize();
            cudaEventRecord(t0, sh);
            cudaStreamWaitEvent(sk, t0, 0);
            std::atomic<int> recorded{0};  // events of this rep recorded so far (no stale-event race)
            std::thread issuer([&] {
                for (int i = 0; i < nch; i++) {
                    while (recorded.load(std::memory_order_acquire) <= i) std::this_thread::yield();
                    cudaEventSynchronize(kk == 2 ? loaded[i] : done[i]);
                    cudaMemcpyAsync(hout + i * chunk, dstage + i * chunk, chunk, cudaMemcpyDeviceToHost, sd);
                }
                cudaEventRecord(td, sd);
            });
            for (int i = 0; i < nch; i++) {
                uint8_t *st = dstage + i * chunk;
                cudaMemcpyAsync(st, hin + i * chunk, chunk, cudaMemcpyHostToDevice, sh);
                cudaEventRecord(loaded[i], sh);
                if (kk < 2) {
                    cudaStreamWaitEvent(sk, loaded[i], 0);
                    if (kk == 0) spin<<<148, 512, 196608, sk>>>(spins[kx]);
                    else touch<<<148, 1024, 0, sk>>>((uint4 *)st, chunk / 16);
                    cudaEventRecord(done[i], sk);
                }
                recorded.store(i + 1, std::memory_order_release);
            }
            cudaEventRecord(th, sh);
            issuer.join();
            cudaDeviceSynchronize();
            float ms, msh;
            cudaEventElapsedTime(&ms, t0, td);
            cudaEventElapsedTime(&msh, t0, th);
            if (ms < best) best = ms, besth = msh;
        }
        const char *nm[] = {"host_issued_d2h_spin", "host_issued_d2h_touch", "host_issued_d2h_no_kernel"};
        printf("{\"variant\": \"%s\", \"spin_ns\": %d, \"chunk_mib\": 16, \"ms\": %.3f, \"gbs\": %.2f, \"h2d_stream_gbs\": %.2f}\n",
               nm[kk], spins[kx], best, total / (best * 1e-3) / 1e9, total / (besth * 1e-3) / 1e9);
    }
    return 0;
}
