/*
 * test_kat.c -- ORACLE self-test binary (test infrastructure only).
 *
 * Usage: test_kat <golden dir>
 * Reads tests/golden/fips197_cipher_kat.txt and sp800_38a_cbc.txt and checks
 * the oracle's Cipher/InvCipher (FIPS-197 App. B, C.1-C.3) and per-page CBC
 * (SP 800-38A F.2.1-F.2.6, as a single 64-byte page) in both directions,
 * plus the exhaustive InvS(S(x)) == x identity.  Exit status 0 = all pass.
 */
#include "kgo_aes.h"

#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static int hex2bin(const char *h, uint8_t *out, int max) {
    int n = (int)strlen(h);
    if (n % 2 || n / 2 > max) return -1;
    for (int i = 0; i < n / 2; i++) {
        unsigned v;
        if (sscanf(h + 2 * i, "%2x", &v) != 1) return -1;
        out[i] = (uint8_t)v;
    }
    return n / 2;
}

static int fails = 0, checks = 0;
static void expect(int ok, const char *what, const char *label) {
    checks++;
    if (!ok) { fails++; fprintf(stderr, "FAIL %s %s\n", what, label); }
}

static FILE *open_golden(const char *dir, const char *name) {
    char path[4096];
    snprintf(path, sizeof path, "%s/%s", dir, name);
    FILE *f = fopen(path, "r");
    if (!f) { fprintf(stderr, "cannot open %s\n", path); exit(2); }
    return f;
}

int main(int argc, char **argv) {
    const char *dir = argc > 1 ? argv[1] : "tests/golden";
    char line[2048], label[64], kh[128], a[512], b[512], c[512];
    kgo_init();

    for (int x = 0; x < 256; x++)
        expect(kgo_inv_sbox(kgo_sbox((uint8_t)x)) == x, "InvS(S(x))", "all x");

    FILE *f = open_golden(dir, "fips197_cipher_kat.txt");
    while (fgets(line, sizeof line, f)) {
        if (line[0] == '#' || line[0] == '\n') continue;
        if (sscanf(line, "%63s %127s %511s %511s", label, kh, a, b) != 4) continue;
        uint8_t key[32], pt[16], ct[16], w[240], got[16];
        int kb = hex2bin(kh, key, 32);
        hex2bin(a, pt, 16);
        hex2bin(b, ct, 16);
        int nr = kgo_key_expansion(key, kb, w);
        kgo_cipher(pt, got, w, nr);
        expect(memcmp(got, ct, 16) == 0, "Cipher", label);
        kgo_inv_cipher(ct, got, w, nr);
        expect(memcmp(got, pt, 16) == 0, "InvCipher", label);
        /* ECB page of one block reproduces the same vector */
        kgo_pages(KGO_ENCRYPT, KGO_MODE_ECB, key, kb, pt, got, 1, 16, NULL, 1);
        expect(memcmp(got, ct, 16) == 0, "ECB page", label);
    }
    fclose(f);

    f = open_golden(dir, "sp800_38a_cbc.txt");
    while (fgets(line, sizeof line, f)) {
        if (line[0] == '#' || line[0] == '\n') continue;
        char ivh[64];
        if (sscanf(line, "%63s %127s %63s %511s %511s", label, kh, ivh, a, c) != 5) continue;
        uint8_t key[32], iv[16], pt[64], ct[64], got[64];
        int kb = hex2bin(kh, key, 32);
        hex2bin(ivh, iv, 16);
        hex2bin(a, pt, 64);
        hex2bin(c, ct, 64);
        kgo_pages(KGO_ENCRYPT, KGO_MODE_CBC, key, kb, pt, got, 1, 64, iv, 1);
        expect(memcmp(got, ct, 64) == 0, "CBC encrypt", label);
        kgo_pages(KGO_DECRYPT, KGO_MODE_CBC, key, kb, ct, got, 1, 64, iv, 1);
        expect(memcmp(got, pt, 64) == 0, "CBC decrypt", label);
        /* in-place */
        memcpy(got, ct, 64);
        kgo_pages(KGO_DECRYPT, KGO_MODE_CBC, key, kb, got, got, 1, 64, iv, 1);
        expect(memcmp(got, pt, 64) == 0, "CBC decrypt in-place", label);
    }
    fclose(f);

    printf("test_kat: %d checks, %d failures\n", checks, fails);
    return fails ? 1 : 0;
}
