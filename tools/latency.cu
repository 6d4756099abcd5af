// latency.cu -- caller-observed latency of one small request through the C ABI
// (no Python): the paper's §3.1 experiment shape ("launch an empty GPU kernel,
// transfer a small amount of input data to it (4KB), and wait for it to
// return ... measured time on the CPU") next to one 4 KiB
// AES-128-CBC decrypt page through kg_submit_pages/kg_wait, HBM- and
// pinned-host-resident.  Prints JSON lines with p10/p50/p90 in microseconds.
//
// build: nvcc -O2 -gencode arch=compute_100a,code=sm_100a tools/latency.cu \
//          -Iinclude -Lpaper_1305_3345_b200 -lkgpu -Xlinker -rpath,'$ORIGIN/../paper_1305_3345_b200' -o build/latency
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#include <algorithm>
#include <vector>

#include "kg.h"

static double now_us() {
    timespec t;
    clock_gettime(CLOCK_MONOTONIC, &t);
    return t.tv_sec * 1e6 + t.tv_nsec * 1e-3;
}

__global__ void empty_kernel(const uint8_t *in) {
    if (threadIdx.x == 1u << 30) printf("%d", in[0]);
}

static void report(const char *name, std::vector<double> &v, int pages) {
    std::sort(v.begin(), v.end());
    size_t n = v.size();
    printf("{\"test\": \"%s\", \"pages\": %d, \"us_p10\": %.2f, \"us_p50\": %.2f, \"us_p90\": %.2f, \"reps\": %zu}\n", name,
           pages, v[n / 10], v[n / 2], v[(9 * n) / 10], n);
}

int main(int argc, char **argv) {
    const int reps = argc > 1 ? atoi(argv[1]) : 2000;
    if (kg_init(0) != KG_OK) {
        fprintf(stderr, "kg_init failed\n");
        return 1;
    }
    uint8_t key[16] = {1, 2, 3};
    kg_set_key(0, key, 16);
    const int PB = 4096;
    uint8_t *d_in, *d_out, *d_iv, *h_in, *h_out, *h_iv;
    cudaMalloc(&d_in, 64 * PB);
    cudaMalloc(&d_out, 64 * PB);
    cudaMalloc(&d_iv, 64 * 16);
    cudaHostAlloc(&h_in, 64 * PB, 0);
    cudaHostAlloc(&h_out, 64 * PB, 0);
    cudaHostAlloc(&h_iv, 64 * 16, 0);
    memset(h_in, 7, 64 * PB);
    memset(h_iv, 1, 64 * 16);
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    std::vector<double> v;

    // paper E1 shape: empty kernel + 4 KB H2D input + wait (traditional launch)
    for (int pass = 0; pass < 2; pass++) {
        v.clear();
        for (int i = 0; i < reps; i++) {
            double t0 = now_us();
            cudaMemcpyAsync(d_in, h_in, PB, cudaMemcpyHostToDevice, st);
            empty_kernel<<<1, 512, 0, st>>>(d_in);
            cudaStreamSynchronize(st);
            v.push_back(now_us() - t0);
        }
    }
    report("empty_kernel_512thr_4KB_h2d_sync", v, 0);

    for (int pages : {1, 2, 16}) {
        for (int pass = 0; pass < 2; pass++) {
            v.clear();
            for (int i = 0; i < reps; i++) {
                double t0 = now_us();
                int64_t t = kg_submit_pages(KG_DECRYPT, KG_MODE_CBC, d_in, d_out, pages, PB, d_iv, 0, st);
                kg_wait(t);
                v.push_back(now_us() - t0);
            }
        }
        report("kg_hbm_dec", v, pages);
        // the same, completion by stream synchronisation instead of kg_wait
        for (int pass = 0; pass < 2; pass++) {
            v.clear();
            for (int i = 0; i < reps; i++) {
                double t0 = now_us();
                int64_t t = kg_submit_pages(KG_DECRYPT, KG_MODE_CBC, d_in, d_out, pages, PB, d_iv, 0, st);
                cudaStreamSynchronize(st);
                v.push_back(now_us() - t0);
                kg_wait(t);
            }
        }
        report("kg_hbm_dec_streamsync", v, pages);
        for (int pass = 0; pass < 2; pass++) {
            v.clear();
            for (int i = 0; i < reps; i++) {
                double t0 = now_us();
                int64_t t = kg_submit_pages(KG_DECRYPT, KG_MODE_CBC, h_in, h_out, pages, PB, h_iv, 0, st);
                kg_wait(t);
                v.push_back(now_us() - t0);
            }
        }
        report("kg_pinned_dec", v, pages);
    }
    // the NSK (row f3): persistent service kernel, requests as messages in pinned memory
    for (int flags : {KG_NSK_DIRECT, 0}) {
        if (kg_nsk_start(16, flags | KG_NSK_NOCAL, 5000) != KG_OK) {
            printf("{\"error\": \"kg_nsk_start failed\"}\n");
            continue;
        }
        for (int pages : {1, 16}) {
            for (int pinned = 0; pinned < 2; pinned++) {
                for (int pass = 0; pass < 2; pass++) {
                    v.clear();
                    for (int i = 0; i < reps; i++) {
                        double t0 = now_us();
                        int64_t t = pinned ? kg_submit_pages(KG_DECRYPT, KG_MODE_CBC, h_in, h_out, pages, PB, h_iv, 0, st)
                                           : kg_submit_pages(KG_DECRYPT, KG_MODE_CBC, d_in, d_out, pages, PB, d_iv, 0, st);
                        kg_wait(t);
                        v.push_back(now_us() - t0);
                    }
                }
                char name[96];
                snprintf(name, sizeof name, "nsk_%s_%s_dec", flags ? "direct" : "ordered", pinned ? "pinned" : "hbm");
                report(name, v, pages);
            }
        }
        kg_nsk_stop();
    }
    // submit-only cost (host side of the request queue)
    v.clear();
    std::vector<int64_t> ts;
    for (int i = 0; i < reps; i++) {
        double t0 = now_us();
        ts.push_back(kg_submit_pages(KG_DECRYPT, KG_MODE_CBC, d_in, d_out, 1, PB, d_iv, 0, st));
        v.push_back(now_us() - t0);
    }
    for (int64_t t : ts) kg_wait(t);
    report("kg_submit_only", v, 1);
    kg_shutdown();
    return 0;
}
