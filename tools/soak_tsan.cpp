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
