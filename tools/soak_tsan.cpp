// soak_tsan.cpp -- host-runtime race check (SURVEY.md §4.2 "TSan on the host
// ticket table"): 4 threads concurrently submit / poll / wait / re-key
// through the C ABI, plus an NSK phase, with the runtime compiled under
// -fsanitize=thread.  Exit 0 = no failures (ThreadSanitizer reports go to
// stderr and make the exit status 66).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <atomic>
#include <thread>
#include <vector>

#include "kg.h"

int main() {
    if (kg_init(0) != KG_OK) return 1;
    const int n = 8, pb = 4096;
    uint8_t *d_in, *d_iv;
    cudaMalloc(&d_in, n * pb);
    cudaMalloc(&d_iv, n * 16);
    cudaMemset(d_in, 3, n * pb);
    uint8_t key[16] = {9};
    for (int k = 0; k < 4; k++) kg_set_key(k, key, 16);
    std::atomic<int> fails{0};
    auto worker = [&](int tid) {
        uint8_t *d_out;
        cudaMalloc(&d_out, n * pb);
        uint8_t k2[16] = {(uint8_t)tid};
        for (int i = 0; i < 300; i++) {
            if (i % 50 == 0) kg_set_key(tid, k2, 16);
            int64_t t = kg_submit_pages(i & 1, 0, d_in, d_out, n, pb, d_iv, tid, nullptr);
            if (t < 0) {
                fails++;
                continue;
            }
            if (i % 3 == 0) kg_poll(t);
            if (kg_wait(t) != KG_OK) fails++;
        }
        cudaFree(d_out);
    };
    // mixed-key and pinned-host (staged) batches from several threads: the
    // key-snapshot ring, the constant-bank key copy, the texture cache and the
    // staging ring are shared state behind the runtime's lock
    auto worker2 = [&](int tid) {
        const int nk = 64;
        uint8_t *h_in = nullptr, *h_out = nullptr, *h_iv = nullptr;
        uint16_t *d_ids = nullptr;
        cudaHostAlloc((void **)&h_in, (size_t)nk * pb, 0);
        cudaHostAlloc((void **)&h_out, (size_t)nk * pb, 0);
        cudaHostAlloc((void **)&h_iv, (size_t)nk * 16, 0);
        cudaMalloc((void **)&d_ids, nk * 2);
        memset(h_in, 5 + tid, (size_t)nk * pb);
        memset(h_iv, 1, (size_t)nk * 16);
        uint16_t ids[nk];
        for (int p = 0; p < nk; p++) ids[p] = (uint16_t)((p + tid) % 4);
        cudaMemcpy(d_ids, ids, sizeof ids, cudaMemcpyHostToDevice);
        uint8_t *d_out2;
        cudaMalloc(&d_out2, (size_t)n * pb);
        for (int i = 0; i < 120; i++) {
            int64_t t;
            if (i % 3 == 0) t = kg_submit_pages(i & 1, 0, h_in, h_out, nk, pb, h_iv, tid, nullptr);  // staged / zero-copy
            else if (i % 3 == 1) t = kg_submit_pages_keyed(i & 1, 1, d_in, d_out2, n, pb, nullptr, d_ids, 16, nullptr);
            else t = kg_submit_pages_keyed(1, 0, h_in, h_out, nk, pb, h_iv, d_ids, 16, nullptr);
            if (t < 0) {
                fails++;
                continue;
            }
            if (kg_wait(t) != KG_OK) fails++;
        }
        cudaFree(d_out2);
        cudaFree(d_ids);
        cudaFreeHost(h_in);
        cudaFreeHost(h_out);
        cudaFreeHost(h_iv);
    };
    {
        kg_set_host_path(KG_HOST_STAGED, 0);
        std::vector<std::thread> th;
        for (int t = 0; t < 4; t++) th.emplace_back(worker2, t);
        for (auto &x : th) x.join();
        kg_set_host_path(KG_HOST_AUTO, 32u << 20);
    }
    for (int phase = 0; phase < 2; phase++) {
        if (phase == 1 && kg_nsk_start(4, KG_NSK_DIRECT, 2000) != KG_OK) return 2;
        std::vector<std::thread> th;
        for (int t = 0; t < 4; t++) th.emplace_back(worker, t);
        for (auto &x : th) x.join();
        if (phase == 1) kg_nsk_stop();
    }
    kg_shutdown();
    printf("soak_tsan: %d failures\n", fails.load());
    return fails.load() ? 1 : 0;
}
