/*
 * kgpu_crypt.c -- a plain-C caller of the C ABI: encrypt or decrypt a file
 * the way an encrypted filesystem treats its pages: 4 KiB
 * pages, one CBC chain per page, a per-page IV (here: the page index as a
 * 16-byte little-endian integer XOR a file IV), AES-128/256.  The file length
 * must be a multiple of 16; a short last page becomes its own 1-page batch.
 *
 *   cc -O2 -Iinclude examples/kgpu_crypt.c -Lpaper_1305_3345_b200 -lkgpu \
 *      -Wl,-rpath,'$ORIGIN/../paper_1305_3345_b200' -o build/kgpu_crypt
 *   build/kgpu_crypt enc 000102...0f <in> <out>     (32 or 64 hex digits)
 *
 * The four steps are the paper's call protocol: get a
 * pinned buffer and fill it (kg_alloc_pinned + read), build and enqueue the
 * request (kg_submit_pages), wait (kg_wait).
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "kg.h"

#define PAGE 4096u

static int hexkey(const char *h, uint8_t *k) {
    size_t n = strlen(h);
    if (n != 32 && n != 64) return -1;
    for (size_t i = 0; i < n / 2; i++) {
        unsigned v;
        if (sscanf(h + 2 * i, "%2x", &v) != 1) return -1;
        k[i] = (uint8_t)v;
    }
    return (int)(n / 2);
}

int main(int argc, char **argv) {
    if (argc != 5 || (strcmp(argv[1], "enc") && strcmp(argv[1], "dec"))) {
        fprintf(stderr, "usage: %s enc|dec <key hex> <in> <out>\n", argv[0]);
        return 2;
    }
    const int dir = strcmp(argv[1], "enc") == 0 ? KG_ENCRYPT : KG_DECRYPT;
    uint8_t key[32];
    const int kb = hexkey(argv[2], key);
    if (kb < 0) {
        fprintf(stderr, "bad key\n");
        return 2;
    }
    FILE *fi = fopen(argv[3], "rb");
    if (!fi) {
        perror(argv[3]);
        return 1;
    }
    fseek(fi, 0, SEEK_END);
    const long len = ftell(fi);
    fseek(fi, 0, SEEK_SET);
    if (len <= 0 || len % 16) {
        fprintf(stderr, "file length must be a positive multiple of 16\n");
        return 1;
    }
    int rc = kg_init(0);
    if (rc != KG_OK) {
        fprintf(stderr, "kg_init: %s\n", kg_strerror(rc));
        return 1;
    }
    if ((rc = kg_set_key(0, key, kb)) != KG_OK) {
        fprintf(stderr, "kg_set_key: %s\n", kg_strerror(rc));
        return 1;
    }
    memset(key, 0, sizeof key); /* the library keeps its own copy */

    const uint64_t full = (uint64_t)len / PAGE, tail = (uint64_t)len % PAGE;
    const uint64_t pages = full + (tail ? 1 : 0);
    uint8_t *buf = (uint8_t *)kg_alloc_pinned((uint64_t)len);
    uint8_t *ivs = (uint8_t *)kg_alloc_pinned(16 * pages);
    if (!buf || !ivs) {
        fprintf(stderr, "kg_alloc_pinned failed\n");
        return 1;
    }
    if (fread(buf, 1, (size_t)len, fi) != (size_t)len) {
        perror("read");
        return 1;
    }
    fclose(fi);
    static const uint8_t file_iv[16] = {0x6b, 0x67, 0x70, 0x75, 0x2d, 0x62, 0x32, 0x30,
                                        0x30, 0x2d, 0x65, 0x78, 0x61, 0x6d, 0x70, 0x6c};
    for (uint64_t p = 0; p < pages; p++)
        for (int b = 0; b < 16; b++) ivs[16 * p + b] = file_iv[b] ^ (uint8_t)(b < 8 ? (p >> (8 * b)) : 0);

    int64_t t1 = -1, t2 = -1;
    if (full) t1 = kg_submit_pages(dir, KG_MODE_CBC, buf, buf, full, PAGE, ivs, 0, NULL);
    if (tail) t2 = kg_submit_pages(dir, KG_MODE_CBC, buf + full * PAGE, buf + full * PAGE, 1, (uint32_t)tail,
                                   ivs + 16 * full, 0, NULL);
    if ((full && t1 < 0) || (tail && t2 < 0)) {
        fprintf(stderr, "kg_submit_pages: %s\n", kg_strerror((int)(t1 < 0 ? t1 : t2)));
        return 1;
    }
    if ((full && (rc = kg_wait(t1)) != KG_OK) || (tail && (rc = kg_wait(t2)) != KG_OK)) {
        fprintf(stderr, "kg_wait: %s\n", kg_strerror(rc));
        return 1;
    }
    FILE *fo = fopen(argv[4], "wb");
    if (!fo || fwrite(buf, 1, (size_t)len, fo) != (size_t)len) {
        perror(argv[4]);
        return 1;
    }
    fclose(fo);
    kg_free_pinned(buf);
    kg_free_pinned(ivs);
    kg_shutdown();
    return 0;
}
