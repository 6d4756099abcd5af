// e1.cu -- the paper's §3.1 launch-overhead experiment (E1) on B200, three arms
// at the paper's three thread counts:
//   "we launch an empty GPU kernel, transfer a small amount of input data to
//    it (4KB), and wait for it to return ... 512 threads 16.7 us, 1024 threads
//    17.3 us, 2048 threads 18.3 us ... the NSK is 1.3x faster".
// Arms (caller-observed, CPU clock, p10/p50/p90 over `reps` after warm-up):
//   launch : cudaMemcpyAsync(4 KB H2D) + empty kernel<<<T threads>>> + cudaStreamSynchronize
//   graph  : the same two operations captured once into a CUDA graph; cudaGraphLaunch + sync
//   nsk    : a persistent kernel of T threads (launched once) polls a doorbell in mapped
//            pinned memory, pulls the 4 KB input over the host link into device memory
//            (zero-copy: the B200 form of "transfer ... to it"), and posts completion to
//            pinned memory; the host rings and spins (the paper's message-based NSK)
// Plus the host-side costs of one kg_submit_pages (pointer classification,
// event record, launch) for DESIGN.md's submit-path breakdown.
// Prints one JSON line per cell.
//
// build: nvcc -O2 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/e1.cu -o build/e1
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#include <algorithm>
#include <atomic>
#include <vector>

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e_ = (x);                                                              \
        if (e_ != cudaSuccess) {                                                           \
            fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
            exit(1);                                                                       \
        }                                                                                  \
    } while (0)

static double now_us() {
    timespec t;
    clock_gettime(CLOCK_MONOTONIC, &t);
    return t.tv_sec * 1e6 + t.tv_nsec * 1e-3;
}

static void report(const char *arm, int threads, std::vector<double> &v, const char *extra = "") {
    std::sort(v.begin(), v.end());
    const size_t n = v.size();
    printf("{\"e1_arm\": \"%s\", \"threads\": %d, \"us_p10\": %.2f, \"us_p50\": %.2f, \"us_p90\": %.2f, \"reps\": %zu%s}\n",
           arm, threads, v[n / 10], v[n / 2], v[(9 * n) / 10], n, extra);
    fflush(stdout);
}

// The "empty" kernel: touches its input so the transfer is not dead.
__global__ void empty_kernel(const uint4 *in, uint4 *sink) {
    if (threadIdx.x == 0x7fffffff) sink[0] = in[0];
}

__global__ void empty_smem_kernel(const uint4 *in, uint4 *sink) {
    extern __shared__ uint4 smem[];
    if (threadIdx.x == 0x7fffffff) sink[0] = smem[in[0].x];
}

// writes 192 KB of shared memory with conflict-free 32-bit stores (the page
// kernels' table-fill traffic, without its global loads)
__global__ void fill_smem_kernel(const uint4 *in, uint4 *sink) {
    extern __shared__ uint32_t sw[];
    for (int i = threadIdx.x; i < 196480 / 4; i += blockDim.x) sw[i] = i;
    __syncthreads();
    if (threadIdx.x == 0x7fffffff) sink[0].x = sw[in[0].x];
}

struct Mailbox {                 // mapped pinned memory
    volatile uint64_t doorbell;  // host -> GPU: request seq
    uint64_t pad0[7];
    volatile uint64_t done;      // GPU -> host: completed seq
    uint64_t pad1[7];
    volatile uint64_t quit;
};

__device__ __forceinline__ uint64_t ld_acquire_sys(const volatile uint64_t *p) {
    uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Persistent "empty service": T threads over ceil(T/1024) CTAs.  Per request:
// CTA 0 thread 0 polls the doorbell; the 4 KB input is read over the host link
// (16 B per thread, 256 threads) into device memory; the CTAs meet at a
// device-scope counter; the last one stores the completion word (system scope).
__global__ void nsk_empty(Mailbox *mb, const uint4 *in_host, uint4 *in_dev, unsigned *arrive, volatile uint64_t *go) {
    for (uint64_t seq = 1;; ++seq) {
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            uint64_t d;
            while ((d = ld_acquire_sys(&mb->doorbell)) < seq) {
                if (mb->quit) break;
            }
            if (mb->quit && d < seq) *go = ~0ull;
            else *go = seq;
            __threadfence();
        }
        if (threadIdx.x == 0)
            while (*go < seq) {
            }
        __syncthreads();
        if (*go == ~0ull) return;
        const unsigned t = blockIdx.x * blockDim.x + threadIdx.x;
        if (t < 256) in_dev[t] = in_host[t];  // the 4 KB "transfer"
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            if (atomicAdd(arrive, 1u) == gridDim.x - 1) {
                *arrive = 0;
                __threadfence_system();
                mb->done = seq;
            }
        }
    }
}

int main(int argc, char **argv) {
    const int reps = argc > 1 ? atoi(argv[1]) : 2000;
    CK(cudaSetDevice(0));
    uint4 *d_in, *d_sink, *h_in;
    CK(cudaMalloc(&d_in, 4096));
    CK(cudaMalloc(&d_sink, 4096));
    CK(cudaHostAlloc(&h_in, 4096, cudaHostAllocMapped));
    memset(h_in, 7, 4096);
    cudaStream_t st;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    std::vector<double> v;

    for (int T : {512, 1024, 2048}) {
        const int tpb = T < 1024 ? T : 1024, grid = T / tpb;
        // ---- launch arm
        for (int pass = 0; pass < 2; pass++) {
            v.clear();
            for (int i = 0; i < reps; i++) {
                const double t0 = now_us();
                cudaMemcpyAsync(d_in, h_in, 4096, cudaMemcpyHostToDevice, st);
                empty_kernel<<<grid, tpb, 0, st>>>(d_in, d_sink);
                cudaStreamSynchronize(st);
                v.push_back(now_us() - t0);
            }
        }
        report("launch", T, v);
        // ---- CUDA graph arm
        cudaGraph_t gr;
        cudaGraphExec_t ge;
        CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal));
        cudaMemcpyAsync(d_in, h_in, 4096, cudaMemcpyHostToDevice, st);
        empty_kernel<<<grid, tpb, 0, st>>>(d_in, d_sink);
        CK(cudaStreamEndCapture(st, &gr));
        CK(cudaGraphInstantiate(&ge, gr, 0));
        for (int pass = 0; pass < 2; pass++) {
            v.clear();
            for (int i = 0; i < reps; i++) {
                const double t0 = now_us();
                cudaGraphLaunch(ge, st);
                cudaStreamSynchronize(st);
                v.push_back(now_us() - t0);
            }
        }
        report("graph", T, v);
        CK(cudaGraphExecDestroy(ge));
        CK(cudaGraphDestroy(gr));
        // ---- NSK arm
        Mailbox *mb, *mb_dev;
        CK(cudaHostAlloc(&mb, sizeof(Mailbox), cudaHostAllocMapped));
        memset((void *)mb, 0, sizeof(Mailbox));
        CK(cudaHostGetDevicePointer((void **)&mb_dev, mb, 0));
        uint4 *h_in_dev;
        CK(cudaHostGetDevicePointer((void **)&h_in_dev, h_in, 0));
        unsigned *arrive;
        uint64_t *go;
        CK(cudaMalloc(&arrive, 4));
        CK(cudaMalloc(&go, 8));
        CK(cudaMemset(arrive, 0, 4));
        CK(cudaMemset(go, 0, 8));
        cudaStream_t ns;
        CK(cudaStreamCreateWithFlags(&ns, cudaStreamNonBlocking));
        void *args[] = {&mb_dev, &h_in_dev, &d_in, &arrive, &go};
        CK(cudaLaunchCooperativeKernel((const void *)nsk_empty, dim3(grid), dim3(tpb), args, 0, ns));
        uint64_t seq = 0;
        for (int pass = 0; pass < 2; pass++) {
            v.clear();
            for (int i = 0; i < reps; i++) {
                const double t0 = now_us();
                ++seq;
                std::atomic_thread_fence(std::memory_order_seq_cst);
                mb->doorbell = seq;
                while (mb->done < seq) {
#if defined(__x86_64__)
                    __builtin_ia32_pause();
#endif
                }
                v.push_back(now_us() - t0);
            }
        }
        report("nsk", T, v);
        mb->quit = 1;
        std::atomic_thread_fence(std::memory_order_seq_cst);
        CK(cudaStreamSynchronize(ns));
        CK(cudaStreamDestroy(ns));
        CK(cudaFree(arrive));
        CK(cudaFree(go));
        CK(cudaFreeHost(mb));
    }

    // ---- launch-latency pieces (no H2D): an empty kernel as is, with the
    // 192 KB dynamic shared memory the page kernels reserve, and with a
    // 192 KB allocation it also fills like the page kernels' table fill
    {
        const int big = 196480;
        CK(cudaFuncSetAttribute(empty_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, big));
        CK(cudaFuncSetAttribute(fill_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, big));
        struct Arm {
            const char *name;
            int which;
        } arms[] = {{"empty_512thr_sync", 0}, {"empty_512thr_192KB_smem_sync", 1}, {"fill_192KB_smem_512thr_sync", 2}};
        for (auto &arm : arms) {
            for (int pass = 0; pass < 2; pass++) {
                v.clear();
                for (int i = 0; i < reps; i++) {
                    const double t0 = now_us();
                    if (arm.which == 0) empty_kernel<<<1, 512, 0, st>>>(d_in, d_sink);
                    else if (arm.which == 1) empty_smem_kernel<<<1, 512, big, st>>>(d_in, d_sink);
                    else fill_smem_kernel<<<1, 512, big, st>>>(d_in, d_sink);
                    cudaStreamSynchronize(st);
                    v.push_back(now_us() - t0);
                }
            }
            report(arm.name, 512, v);
        }
    }

    // ---- host-side pieces of a submit (for the submit-path breakdown)
    {
        cudaPointerAttributes at;
        cudaEvent_t ev;
        CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        struct Item {
            const char *name;
            int which;
        } items[] = {{"cudaPointerGetAttributes(device)", 0}, {"cudaPointerGetAttributes(pinned)", 1},
                     {"cudaGetDevice", 2}, {"cudaEventRecord", 3}, {"empty launch (no sync)", 4}};
        for (auto &it : items) {
            const int n = 20000;
            int dev;
            const double t0 = now_us();
            for (int i = 0; i < n; i++) {
                switch (it.which) {
                    case 0: cudaPointerGetAttributes(&at, d_in); break;
                    case 1: cudaPointerGetAttributes(&at, h_in); break;
                    case 2: cudaGetDevice(&dev); break;
                    case 3: cudaEventRecord(ev, st); break;
                    case 4: empty_kernel<<<1, 512, 0, st>>>(d_in, d_sink); break;
                }
            }
            const double per = (now_us() - t0) / n;
            cudaStreamSynchronize(st);
            printf("{\"host_cost\": \"%s\", \"us\": %.3f}\n", it.name, per);
        }
    }
    return 0;
}
