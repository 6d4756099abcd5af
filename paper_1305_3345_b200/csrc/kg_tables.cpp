// kg_tables.cpp -- GPU-path host code: the S-box, the T-table bases and the
// key schedules.  Written independently of oracle/: the S-box inverse here is
// x^254 by square-and-multiply over a carry-less product reduced by long
// division (the oracle uses log/antilog tables), the affine map is the
// rotate form, and everything is word-oriented little-endian.
//
// FIPS-197 §5.1.1 (S-box), §5.1.3 / §5.3.3 (MixColumns / InvMixColumns
// coefficients that the T-tables fold in), §5.2 (KeyExpansion), §5.3.5
// (equivalent inverse cipher key schedule).  The paper itself only says it
// "implemented the AES encryption algorithm as a service".
#include <string.h>

#include "kg_internal.h"

namespace kg {
namespace {

// GF(2^8) product: 15-bit carry-less product, then reduce modulo
// m(x) = x^8 + x^4 + x^3 + x + 1 (0x11b) from the top bit down.
uint8_t gmul(uint8_t a, uint8_t b) {
    uint32_t p = 0;
    for (int i = 0; i < 8; i++)
        if (b & (1u << i)) p ^= (uint32_t)a << i;
    for (int bit = 14; bit >= 8; bit--)
        if (p & (1u << bit)) p ^= 0x11bu << (bit - 8);
    return (uint8_t)p;
}

// a^254 = a^-1 for a != 0 (and 0 -> 0): square-and-multiply over 254 = 0b11111110.
uint8_t ginv(uint8_t a) {
    uint8_t result = 1, base = a;
    unsigned e = 254;
    while (e) {
        if (e & 1) result = gmul(result, base);
        base = gmul(base, base);
        e >>= 1;
    }
    return a ? result : 0;
}

inline uint8_t rotl8(uint8_t x, int s) { return (uint8_t)((x << s) | (x >> (8 - s))); }

uint8_t sbox_of(uint8_t x) {
    uint8_t b = ginv(x);
    return (uint8_t)(b ^ rotl8(b, 1) ^ rotl8(b, 2) ^ rotl8(b, 3) ^ rotl8(b, 4) ^ 0x63);
}

struct Sboxes {
    uint8_t s[256], si[256];
    Sboxes() {
        for (int x = 0; x < 256; x++) s[x] = sbox_of((uint8_t)x);
        for (int x = 0; x < 256; x++) si[s[x]] = (uint8_t)x;
    }
};

const Sboxes &sboxes() {
    static const Sboxes S;
    return S;
}

inline uint32_t sub_word(uint32_t w) {
    const uint8_t *s = sboxes().s;
    return (uint32_t)s[w & 0xff] | ((uint32_t)s[(w >> 8) & 0xff] << 8) |
           ((uint32_t)s[(w >> 16) & 0xff] << 16) | ((uint32_t)s[w >> 24] << 24);
}

// InvMixColumns of one column word (LE: byte r = row r).
uint32_t inv_mix_word(uint32_t w) {
    uint8_t a[4], o[4];
    for (int r = 0; r < 4; r++) a[r] = (uint8_t)(w >> (8 * r));
    static const uint8_t M[4][4] = {{14, 11, 13, 9}, {9, 14, 11, 13}, {13, 9, 14, 11}, {11, 13, 9, 14}};
    for (int r = 0; r < 4; r++) {
        o[r] = 0;
        for (int k = 0; k < 4; k++) o[r] ^= gmul(M[r][k], a[k]);
    }
    return (uint32_t)o[0] | ((uint32_t)o[1] << 8) | ((uint32_t)o[2] << 16) | ((uint32_t)o[3] << 24);
}

}  // namespace

void build_base_tables(BaseTables *t) {
    const Sboxes &S = sboxes();
    for (int x = 0; x < 256; x++) {
        uint8_t s = S.s[x], si = S.si[x];
        t->te0[x] = (uint32_t)gmul(s, 2) | ((uint32_t)s << 8) | ((uint32_t)s << 16) | ((uint32_t)gmul(s, 3) << 24);
        t->td0[x] = (uint32_t)gmul(si, 14) | ((uint32_t)gmul(si, 9) << 8) | ((uint32_t)gmul(si, 13) << 16) |
                    ((uint32_t)gmul(si, 11) << 24);
        t->isb4[x] = (uint32_t)si * 0x01010101u;
    }
}

int expand_key(const uint8_t *key, int key_bytes, RoundKeys *enc, RoundKeys *dec) {
    int nk;
    switch (key_bytes) {
        case 16: nk = 4; break;
        case 24: nk = 6; break;
        case 32: nk = 8; break;
        default: return -1;
    }
    const int nr = nk + 6;
    const int total = 4 * (nr + 1);
    uint32_t w[60];
    for (int i = 0; i < nk; i++)
        w[i] = (uint32_t)key[4 * i] | ((uint32_t)key[4 * i + 1] << 8) | ((uint32_t)key[4 * i + 2] << 16) |
               ((uint32_t)key[4 * i + 3] << 24);
    uint8_t rc = 1;
    for (int i = nk; i < total; i++) {
        uint32_t t = w[i - 1];
        if (i % nk == 0) {
            t = sub_word((t >> 8) | (t << 24)) ^ rc;  // RotWord is a right rotate of the LE word
            rc = gmul(rc, 2);
        } else if (nk == 8 && i % nk == 4) {
            t = sub_word(t);
        }
        w[i] = w[i - nk] ^ t;
    }
    memset(enc, 0, sizeof *enc);
    memset(dec, 0, sizeof *dec);
    for (int i = 0; i < total; i++) enc->w[i] = w[i];
    for (int r = 0; r <= nr; r++)
        for (int c = 0; c < 4; c++) {
            uint32_t x = w[4 * (nr - r) + c];
            dec->w[4 * r + c] = (r == 0 || r == nr) ? x : inv_mix_word(x);
        }
    return nr;
}

}  // namespace kg
