/*
 * kgo_aes.h -- the ORACLE: a plain, slow, obviously-correct CPU AES.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load or execute
 * anything under oracle/.  The product (paper_1305_3345_b200/) never
 * links, imports or calls it, and shares no code, header, table or
 * generator with it.
 *
 * What it computes (exactly, one correct output):
 *   - FIPS-197 AES (§5.1 Cipher, §5.2 KeyExpansion, §5.3 InvCipher --
 *     the *straightforward* inverse cipher, not the §5.3.5 equivalent
 *     form the GPU path uses) for Nk = 4/6/8 (AES-128/192/256).
 *   - NIST SP 800-38A §6.2 CBC, one chain per page with a per-page IV,
 *     over a batch of contiguous pages [n_pages][page_bytes].
 *   - ECB pages (the paper's own mode, §3.3) for the
 *     NEXT-f1 row.
 *
 * Paper passages: AES offloaded as a GPU service for the Linux crypto
 * subsystem (§3.3); decryption exists and "has similar
 * performance" (Fig. 2 caption); per-page use by
 * encrypted filesystems.  CBC per page + per-page IV
 * is the north star's reading (BASELINE.json:5).
 *
 * Construction rules: C99, no intrinsics, byte
 * oriented, S-box computed at init from its GF(2^8) definition via
 * log/antilog tables with generator 0x03 (FIPS-197 §4.2, §5.1.1).
 *
 * Parity status: every function below is pinned by tests under tests/
 * (FIPS-197 App. A/B/C, SP 800-38A F.2.1-F.2.6, GF spot values, S-box
 * spot values, InvS o S = id, OpenSSL cross-check, CBC identities).
 */
#ifndef KGO_AES_H
#define KGO_AES_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Build the S-box / inverse S-box (idempotent, thread-safe after the first
 * call returns; kgo_cbc_pages calls it before spawning threads). */
void kgo_init(void);

/* FIPS-197 §4.2 multiplication in GF(2^8) mod x^8+x^4+x^3+x+1. */
uint8_t kgo_gf_mul(uint8_t a, uint8_t b);
/* FIPS-197 §4.2.1 xtime(). */
uint8_t kgo_xtime(uint8_t a);
/* FIPS-197 §5.1.1 S-box and its inverse (§5.3.2). */
uint8_t kgo_sbox(uint8_t x);
uint8_t kgo_inv_sbox(uint8_t x);

/* The individual round transformations on a 16-byte state laid out as
 * in[] (FIPS-197 §3.4: s[r][c] = in[r + 4c]); exposed for step pins
 * against FIPS-197 Appendix B. */
void kgo_sub_bytes(uint8_t s[16]);
void kgo_shift_rows(uint8_t s[16]);
void kgo_mix_columns(uint8_t s[16]);
void kgo_inv_sub_bytes(uint8_t s[16]);
void kgo_inv_shift_rows(uint8_t s[16]);
void kgo_inv_mix_columns(uint8_t s[16]);
void kgo_add_round_key(uint8_t s[16], const uint8_t *w_round /* 16 bytes */);

/* FIPS-197 §5.2 KeyExpansion.  key_bytes in {16,24,32}.  w receives
 * 4*(Nr+1) words as bytes (w[4i..4i+3] = word i, byte 0 = most significant
 * in the standard's hex notation), i.e. 176/208/240 bytes.
 * Returns Nr, or -1 on a bad key length. */
int kgo_key_expansion(const uint8_t *key, int key_bytes, uint8_t *w);

/* FIPS-197 §5.1 Cipher and §5.3 InvCipher on one 16-byte block. */
void kgo_cipher(const uint8_t in[16], uint8_t out[16], const uint8_t *w, int nr);
void kgo_inv_cipher(const uint8_t in[16], uint8_t out[16], const uint8_t *w, int nr);

/* Directions / modes, numerically equal to the product ABI's values so a
 * test can pass the same integers to both (the values are a convention,
 * not shared code). */
#define KGO_ENCRYPT 0
#define KGO_DECRYPT 1
#define KGO_MODE_CBC 0
#define KGO_MODE_ECB 1

/* SP 800-38A §6.2 CBC (mode 0) or §6.1 ECB (mode 1) over n_pages pages of
 * page_bytes each, one chain per page, page p's IV at ivs[16p] (ignored for
 * ECB, may be NULL).  in == out (exact alias) is allowed.  Pages are split
 * into contiguous ranges over `threads` pthreads (threads <= 1: caller's
 * thread).  Returns 0, or -1 on bad arguments (page_bytes % 16 != 0, zero
 * sizes, bad key). */
int kgo_pages(int dir, int mode, const uint8_t *key, int key_bytes,
              const uint8_t *in, uint8_t *out, uint64_t n_pages,
              uint32_t page_bytes, const uint8_t *ivs, int threads);

#ifdef __cplusplus
}
#endif
#endif
