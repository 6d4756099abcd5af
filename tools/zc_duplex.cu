// zc_duplex.cu -- can SM-issued host-memory traffic (zero-copy loads/stores
// over the host link) replace one copy engine of the staged pinned pipeline?
// 256 MiB each way, pinned + mapped host buffers, CUDA-event timed, best of 5:
//   ce_h2d, ce_d2h, ce_duplex      : copy engines alone / both at once
//   sm_write, sm_read              : a 148 x 1024 kernel storing to / loading from host memory
//   ce_h2d + sm_write              : H2D copy engine while a kernel writes the other direction
//   sm_read + ce_d2h               : kernel reads host memory while the D2H engine runs
// One JSON line per arm (GB/s per direction).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#define CK(x)                                                                               \
    do {                                                                                    \
        cudaError_t e_ = (x);                                                               \
        if (e_ != cudaSuccess) {                                                            \
            fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
            return 1;                                                                       \
        }                                                                                   \
    } while (0)

__global__ void copy_kernel(const uint4 *__restrict__ src, uint4 *__restrict__ dst, size_t n) {
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (; i < n; i += stride) dst[i] = src[i];
}

int main() {
    const size_t bytes = 256ull << 20, n = bytes / 16;
    uint8_t *h_a, *h_b, *d_a, *d_b, *d_c, *d_d;
    CK(cudaHostAlloc(&h_a, bytes, cudaHostAllocMapped));
    CK(cudaHostAlloc(&h_b, bytes, cudaHostAllocMapped));
    memset(h_a, 1, bytes);
    memset(h_b, 2, bytes);
    CK(cudaMalloc(&d_a, bytes));
    CK(cudaMalloc(&d_b, bytes));
    CK(cudaMalloc(&d_c, bytes));
    CK(cudaMalloc(&d_d, bytes));
    uint8_t *h_a_dev, *h_b_dev;
    CK(cudaHostGetDevicePointer((void **)&h_a_dev, h_a, 0));
    CK(cudaHostGetDevicePointer((void **)&h_b_dev, h_b, 0));
    cudaStream_t s1, s2;
    CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
    cudaEvent_t e0, e1a, e1b;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1a));
    CK(cudaEventCreate(&e1b));
    const int grid = 148 * 2, tpb = 1024;

    // arm: 0 ce_h2d, 1 ce_d2h, 2 sm_write, 3 sm_read
    auto issue = [&](int op, cudaStream_t st) {
        switch (op) {
            case 0: cudaMemcpyAsync(d_a, h_a, bytes, cudaMemcpyHostToDevice, st); break;
            case 1: cudaMemcpyAsync(h_b, d_b, bytes, cudaMemcpyDeviceToHost, st); break;
            case 2: copy_kernel<<<grid, tpb, 0, st>>>((const uint4 *)d_c, (uint4 *)h_b_dev, n); break;
            case 3: copy_kernel<<<grid, tpb, 0, st>>>((const uint4 *)h_a_dev, (uint4 *)d_d, n); break;
        }
    };
    const char *names[] = {"ce_h2d", "ce_d2h", "sm_write_to_host", "sm_read_from_host"};
    struct Arm {
        int a, b;  // b < 0: alone
    } arms[] = {{0, -1}, {1, -1}, {2, -1}, {3, -1}, {0, 1}, {0, 2}, {3, 1}, {3, 2}};
    for (auto &arm : arms) {
        double best_a = 1e30, best_b = 1e30;
        for (int rep = 0; rep < 6; rep++) {
            CK(cudaDeviceSynchronize());
            CK(cudaEventRecord(e0, s1));
            CK(cudaStreamWaitEvent(s2, e0, 0));
            issue(arm.a, s1);
            CK(cudaEventRecord(e1a, s1));
            if (arm.b >= 0) {
                issue(arm.b, s2);
                CK(cudaEventRecord(e1b, s2));
            }
            CK(cudaDeviceSynchronize());
            float ta = 0, tb = 0;
            CK(cudaEventElapsedTime(&ta, e0, e1a));
            if (arm.b >= 0) CK(cudaEventElapsedTime(&tb, e0, e1b));
            if (rep == 0) continue;  // warm-up
            best_a = ta < best_a ? ta : best_a;
            if (arm.b >= 0) best_b = tb < best_b ? tb : best_b;
        }
        if (arm.b < 0)
            printf("{\"arm\": \"%s\", \"gbs\": %.2f}\n", names[arm.a], bytes / (best_a * 1e-3) / 1e9);
        else
            printf("{\"arm\": \"%s + %s\", \"gbs_first\": %.2f, \"gbs_second\": %.2f}\n", names[arm.a], names[arm.b],
                   bytes / (best_a * 1e-3) / 1e9, bytes / (best_b * 1e-3) / 1e9);
        fflush(stdout);
    }
    return 0;
}
