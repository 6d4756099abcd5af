/*
 * kgo_aes.c -- ORACLE (test infrastructure only; see kgo_aes.h header).
 *
 * FIPS-197 AES written out step by step in the standard's order and
 * notation.  Byte oriented; the state is s[r][c] = in[r + 4c] (FIPS-197
 * §3.4), stored as the 16-byte array in[] itself, so state[r][c] is
 * st[r + 4*c].  No tables beyond the S-box (computed at init from its
 * definition) and the GF(2^8) log/antilog tables used to compute it.
 *
 * The paper offloads "the AES encryption algorithm as a service"
 * (§3.3); it gives no algorithmic detail, so the
 * definition is FIPS-197's.
 */
#include "kgo_aes.h"

#include <string.h>

static uint8_t sbox_tab[256];
static uint8_t inv_sbox_tab[256];
static volatile int sbox_ready = 0;

/* ---- FIPS-197 §4.2: arithmetic in GF(2^8) ------------------------------ */

/* §4.2.1: multiplication by x, i.e. {02}; reduce by m(x) = {01}{1b}. */
uint8_t kgo_xtime(uint8_t a) {
    return (uint8_t)((a << 1) ^ ((a & 0x80) ? 0x1b : 0x00));
}

/* §4.2: general product by repeated xtime() over the bits of b
 * ("multiplication by higher powers of x can be implemented by repeated
 * application of xtime()"). */
uint8_t kgo_gf_mul(uint8_t a, uint8_t b) {
    uint8_t acc = 0;
    while (b) {
        if (b & 1) acc ^= a;
        a = kgo_xtime(a);
        b >>= 1;
    }
    return acc;
}

/* ---- FIPS-197 §5.1.1: the S-box from its definition -------------------- */
/* 1. multiplicative inverse in GF(2^8) ({00} maps to itself), computed with
 *    log/antilog tables for the generator {03};
 * 2. the affine transformation
 *    b'_i = b_i ^ b_(i+4)%8 ^ b_(i+5)%8 ^ b_(i+6)%8 ^ b_(i+7)%8 ^ c_i,
 *    c = {63}, written bit by bit as in equation (5.1). */
static void build_sbox(void) {
    uint8_t alog[256], lg[256];
    uint8_t v = 1;
    memset(lg, 0, sizeof lg);
    for (int i = 0; i < 255; i++) {
        alog[i] = v;
        lg[v] = (uint8_t)i;
        v = kgo_gf_mul(v, 0x03);
    }
    alog[255] = alog[0];
    for (int x = 0; x < 256; x++) {
        uint8_t inv = (x == 0) ? 0 : alog[(255 - lg[x]) % 255];
        uint8_t out = 0;
        for (int i = 0; i < 8; i++) {
            int bit = ((inv >> i) & 1) ^ ((inv >> ((i + 4) % 8)) & 1) ^
                      ((inv >> ((i + 5) % 8)) & 1) ^ ((inv >> ((i + 6) % 8)) & 1) ^
                      ((inv >> ((i + 7) % 8)) & 1) ^ ((0x63 >> i) & 1);
            out |= (uint8_t)(bit << i);
        }
        sbox_tab[x] = out;
    }
    /* §5.3.2: InvSubBytes uses the inverse of the S-box. */
    for (int x = 0; x < 256; x++) inv_sbox_tab[sbox_tab[x]] = (uint8_t)x;
}

void kgo_init(void) {
    if (!sbox_ready) {
        build_sbox();
        sbox_ready = 1;
    }
}

uint8_t kgo_sbox(uint8_t x) { kgo_init(); return sbox_tab[x]; }
uint8_t kgo_inv_sbox(uint8_t x) { kgo_init(); return inv_sbox_tab[x]; }

/* ---- FIPS-197 §5.1: Cipher transformations ----------------------------- */
#define ST(s, r, c) ((s)[(r) + 4 * (c)])

/* §5.1.1 SubBytes */
void kgo_sub_bytes(uint8_t s[16]) {
    kgo_init();
    for (int i = 0; i < 16; i++) s[i] = sbox_tab[s[i]];
}

/* §5.1.2 ShiftRows: s'[r][c] = s[r][(c + shift(r,4)) mod 4], shift(r,4)=r */
void kgo_shift_rows(uint8_t s[16]) {
    uint8_t t[16];
    for (int r = 0; r < 4; r++)
        for (int c = 0; c < 4; c++) ST(t, r, c) = ST(s, r, (c + r) % 4);
    memcpy(s, t, 16);
}

/* §5.1.3 MixColumns, equation (5.6):
 *   s'0 = ({02}•s0) ^ ({03}•s1) ^ s2 ^ s3
 *   s'1 = s0 ^ ({02}•s1) ^ ({03}•s2) ^ s3
 *   s'2 = s0 ^ s1 ^ ({02}•s2) ^ ({03}•s3)
 *   s'3 = ({03}•s0) ^ s1 ^ s2 ^ ({02}•s3)                               */
void kgo_mix_columns(uint8_t s[16]) {
    for (int c = 0; c < 4; c++) {
        uint8_t a0 = ST(s, 0, c), a1 = ST(s, 1, c), a2 = ST(s, 2, c), a3 = ST(s, 3, c);
        ST(s, 0, c) = (uint8_t)(kgo_gf_mul(0x02, a0) ^ kgo_gf_mul(0x03, a1) ^ a2 ^ a3);
        ST(s, 1, c) = (uint8_t)(a0 ^ kgo_gf_mul(0x02, a1) ^ kgo_gf_mul(0x03, a2) ^ a3);
        ST(s, 2, c) = (uint8_t)(a0 ^ a1 ^ kgo_gf_mul(0x02, a2) ^ kgo_gf_mul(0x03, a3));
        ST(s, 3, c) = (uint8_t)(kgo_gf_mul(0x03, a0) ^ a1 ^ a2 ^ kgo_gf_mul(0x02, a3));
    }
}

/* §5.1.4 AddRoundKey: column c XOR word w[round*Nb + c]; w_round points at
 * the 16 bytes of the round's four words (byte j of word c = row j). */
void kgo_add_round_key(uint8_t s[16], const uint8_t *w_round) {
    for (int c = 0; c < 4; c++)
        for (int r = 0; r < 4; r++) ST(s, r, c) ^= w_round[4 * c + r];
}

/* ---- FIPS-197 §5.3: InvCipher transformations -------------------------- */

/* §5.3.1 InvShiftRows: s'[r][(c + shift(r,4)) mod 4] = s[r][c] */
void kgo_inv_shift_rows(uint8_t s[16]) {
    uint8_t t[16];
    for (int r = 0; r < 4; r++)
        for (int c = 0; c < 4; c++) ST(t, r, (c + r) % 4) = ST(s, r, c);
    memcpy(s, t, 16);
}

/* §5.3.2 InvSubBytes */
void kgo_inv_sub_bytes(uint8_t s[16]) {
    kgo_init();
    for (int i = 0; i < 16; i++) s[i] = inv_sbox_tab[s[i]];
}

/* §5.3.3 InvMixColumns, equation (5.10):
 *   s'0 = {0e}•s0 ^ {0b}•s1 ^ {0d}•s2 ^ {09}•s3
 *   s'1 = {09}•s0 ^ {0e}•s1 ^ {0b}•s2 ^ {0d}•s3
 *   s'2 = {0d}•s0 ^ {09}•s1 ^ {0e}•s2 ^ {0b}•s3
 *   s'3 = {0b}•s0 ^ {0d}•s1 ^ {09}•s2 ^ {0e}•s3                         */
void kgo_inv_mix_columns(uint8_t s[16]) {
    for (int c = 0; c < 4; c++) {
        uint8_t a0 = ST(s, 0, c), a1 = ST(s, 1, c), a2 = ST(s, 2, c), a3 = ST(s, 3, c);
        ST(s, 0, c) = (uint8_t)(kgo_gf_mul(0x0e, a0) ^ kgo_gf_mul(0x0b, a1) ^
                                kgo_gf_mul(0x0d, a2) ^ kgo_gf_mul(0x09, a3));
        ST(s, 1, c) = (uint8_t)(kgo_gf_mul(0x09, a0) ^ kgo_gf_mul(0x0e, a1) ^
                                kgo_gf_mul(0x0b, a2) ^ kgo_gf_mul(0x0d, a3));
        ST(s, 2, c) = (uint8_t)(kgo_gf_mul(0x0d, a0) ^ kgo_gf_mul(0x09, a1) ^
                                kgo_gf_mul(0x0e, a2) ^ kgo_gf_mul(0x0b, a3));
        ST(s, 3, c) = (uint8_t)(kgo_gf_mul(0x0b, a0) ^ kgo_gf_mul(0x0d, a1) ^
                                kgo_gf_mul(0x09, a2) ^ kgo_gf_mul(0x0e, a3));
    }
}

/* ---- FIPS-197 §5.2: KeyExpansion (Fig. 11) ------------------------------ */
int kgo_key_expansion(const uint8_t *key, int key_bytes, uint8_t *w) {
    int nk, nr;
    kgo_init();
    switch (key_bytes) {
        case 16: nk = 4; nr = 10; break;
        case 24: nk = 6; nr = 12; break;
        case 32: nk = 8; nr = 14; break;
        default: return -1;
    }
    const int nb = 4;
    /* w[i] = word(key[4i], key[4i+1], key[4i+2], key[4i+3]) for i < Nk */
    for (int i = 0; i < 4 * nk; i++) w[i] = key[i];
    uint8_t rcon = 0x01; /* Rcon[i/Nk] = [x^(i/Nk - 1), {00}, {00}, {00}] */
    for (int i = nk; i < nb * (nr + 1); i++) {
        uint8_t temp[4];
        memcpy(temp, &w[4 * (i - 1)], 4);
        if (i % nk == 0) {
            /* temp = SubWord(RotWord(temp)) xor Rcon[i/Nk] */
            uint8_t t0 = temp[0];
            temp[0] = temp[1]; temp[1] = temp[2]; temp[2] = temp[3]; temp[3] = t0;
            for (int k = 0; k < 4; k++) temp[k] = sbox_tab[temp[k]];
            temp[0] ^= rcon;
            rcon = kgo_xtime(rcon);
        } else if (nk > 6 && i % nk == 4) {
            /* temp = SubWord(temp) */
            for (int k = 0; k < 4; k++) temp[k] = sbox_tab[temp[k]];
        }
        for (int k = 0; k < 4; k++) w[4 * i + k] = (uint8_t)(w[4 * (i - nk) + k] ^ temp[k]);
    }
    return nr;
}

/* ---- FIPS-197 §5.1 Cipher (Fig. 5) -------------------------------------- */
void kgo_cipher(const uint8_t in[16], uint8_t out[16], const uint8_t *w, int nr) {
    uint8_t s[16];
    memcpy(s, in, 16);
    kgo_add_round_key(s, &w[0]);
    for (int round = 1; round <= nr - 1; round++) {
        kgo_sub_bytes(s);
        kgo_shift_rows(s);
        kgo_mix_columns(s);
        kgo_add_round_key(s, &w[16 * round]);
    }
    kgo_sub_bytes(s);
    kgo_shift_rows(s);
    kgo_add_round_key(s, &w[16 * nr]);
    memcpy(out, s, 16);
}

/* ---- FIPS-197 §5.3 InvCipher (Fig. 12) ---------------------------------- */
void kgo_inv_cipher(const uint8_t in[16], uint8_t out[16], const uint8_t *w, int nr) {
    uint8_t s[16];
    memcpy(s, in, 16);
    kgo_add_round_key(s, &w[16 * nr]);
    for (int round = nr - 1; round >= 1; round--) {
        kgo_inv_shift_rows(s);
        kgo_inv_sub_bytes(s);
        kgo_add_round_key(s, &w[16 * round]);
        kgo_inv_mix_columns(s);
    }
    kgo_inv_shift_rows(s);
    kgo_inv_sub_bytes(s);
    kgo_add_round_key(s, &w[0]);
    memcpy(out, s, 16);
}
