/*
 * kgo_pages.c -- ORACLE (test infrastructure only; see kgo_aes.h header).
 *
 * NIST SP 800-38A modes applied page by page, written as the standard
 * states them:
 *   §6.2 CBC Encryption: C_1 = CIPH_K(P_1 ^ IV);  C_j = CIPH_K(P_j ^ C_{j-1})
 *        CBC Decryption: P_1 = CIPH^-1_K(C_1) ^ IV; P_j = CIPH^-1_K(C_j) ^ C_{j-1}
 *   §6.1 ECB: C_j = CIPH_K(P_j);  P_j = CIPH^-1_K(C_j)
 * with one chain per page and page p's IV at ivs[16p] (BASELINE.json:5:
 * "one CBC chain per page with a per-page IV"; readings R1-R4).
 * Pages are independent, so a pthread split over contiguous page ranges
 * changes nothing but wall time.
 *
 * Aliasing: in == out is allowed.  The decryptor keeps the previous
 * *ciphertext* block in a local copy before overwriting it, exactly the
 * C_{j-1} of the formula.
 */
#include "kgo_aes.h"

#include <pthread.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    int dir, mode, nr;
    const uint8_t *w;
    const uint8_t *in;
    uint8_t *out;
    uint64_t p0, p1;
    uint32_t page_bytes;
    const uint8_t *ivs;
} kgo_job;

static void one_page(const kgo_job *j, uint64_t p) {
    const uint8_t *in = j->in + p * (uint64_t)j->page_bytes;
    uint8_t *out = j->out + p * (uint64_t)j->page_bytes;
    const uint32_t nblk = j->page_bytes / 16;
    uint8_t prev[16], x[16], y[16];
    if (j->mode == KGO_MODE_CBC) memcpy(prev, j->ivs + 16 * p, 16); /* C_0 := IV */
    for (uint32_t b = 0; b < nblk; b++) {
        memcpy(x, in + 16 * (uint64_t)b, 16);
        if (j->mode == KGO_MODE_ECB) {
            if (j->dir == KGO_ENCRYPT) kgo_cipher(x, y, j->w, j->nr);
            else kgo_inv_cipher(x, y, j->w, j->nr);
        } else if (j->dir == KGO_ENCRYPT) {
            /* C_j = CIPH_K(P_j xor C_{j-1}) */
            for (int k = 0; k < 16; k++) x[k] ^= prev[k];
            kgo_cipher(x, y, j->w, j->nr);
            memcpy(prev, y, 16);
        } else {
            /* P_j = CIPH^-1_K(C_j) xor C_{j-1} */
            kgo_inv_cipher(x, y, j->w, j->nr);
            for (int k = 0; k < 16; k++) y[k] ^= prev[k];
            memcpy(prev, x, 16);
        }
        memcpy(out + 16 * (uint64_t)b, y, 16);
    }
}

static void *run_range(void *arg) {
    const kgo_job *j = (const kgo_job *)arg;
    for (uint64_t p = j->p0; p < j->p1; p++) one_page(j, p);
    return NULL;
}

int kgo_pages(int dir, int mode, const uint8_t *key, int key_bytes,
              const uint8_t *in, uint8_t *out, uint64_t n_pages,
              uint32_t page_bytes, const uint8_t *ivs, int threads) {
    uint8_t w[240];
    if ((dir != KGO_ENCRYPT && dir != KGO_DECRYPT) ||
        (mode != KGO_MODE_CBC && mode != KGO_MODE_ECB))
        return -1;
    if (n_pages == 0 || page_bytes == 0 || page_bytes % 16 != 0) return -1;
    if (!key || !in || !out || (mode == KGO_MODE_CBC && !ivs)) return -1;
    kgo_init();
    int nr = kgo_key_expansion(key, key_bytes, w);
    if (nr < 0) return -1;
    if (threads < 1) threads = 1;
    if ((uint64_t)threads > n_pages) threads = (int)n_pages;

    kgo_job *jobs = (kgo_job *)calloc((size_t)threads, sizeof(kgo_job));
    pthread_t *tids = (pthread_t *)calloc((size_t)threads, sizeof(pthread_t));
    if (!jobs || !tids) { free(jobs); free(tids); return -1; }
    for (int t = 0; t < threads; t++) {
        jobs[t].dir = dir; jobs[t].mode = mode; jobs[t].nr = nr; jobs[t].w = w;
        jobs[t].in = in; jobs[t].out = out; jobs[t].page_bytes = page_bytes;
        jobs[t].ivs = ivs;
        jobs[t].p0 = n_pages * (uint64_t)t / (uint64_t)threads;
        jobs[t].p1 = n_pages * (uint64_t)(t + 1) / (uint64_t)threads;
    }
    if (threads == 1) {
        run_range(&jobs[0]);
    } else {
        int started = 0;
        for (int t = 1; t < threads; t++) {
            if (pthread_create(&tids[t], NULL, run_range, &jobs[t]) != 0) break;
            started = t;
        }
        run_range(&jobs[0]);
        for (int t = 1; t <= started; t++) pthread_join(tids[t], NULL);
        /* any range whose thread failed to start runs here */
        for (int t = started + 1; t < threads; t++) run_range(&jobs[t]);
    }
    free(jobs);
    free(tids);
    return 0;
}
