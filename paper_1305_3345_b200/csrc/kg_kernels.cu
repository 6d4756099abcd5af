// kg_kernels.cu -- the AES page kernels for sm_100a.
//
// What they compute (exactly, bit for bit): FIPS-197 AES over 16-byte
// blocks, chained per page as NIST SP 800-38A §6.2 CBC (one chain per page,
// per-page IV, BASELINE.json:5) or §6.1 ECB (the paper's mode).
// Decryption uses the equivalent inverse cipher (FIPS-197 §5.3.5) with the
// schedule kg_tables.cpp prepares.
//
// B200 design:
//  * The bound is the shared-memory data path (32 lane-lookups/clk/SM), not
//    HBM and not tensor cores: 16 table lookups per block-round.
//  * T-tables live in shared memory replicated 32x so that lane l only ever
//    touches bank l (conflict-free by construction).  Entry x of table i
//    for lane l sits at byte  (i>>1)*64K + x*256 + (i&1)*128 + l*4.  One
//    PRMT (__byte_perm) turns (state word, lane bytes) into that offset, so a
//    lookup is exactly PRMT + LDS; the region base is an LDS immediate.
//  * Round keys come by value in the kernel parameter (constant bank), so
//    AddRoundKey folds into the 3-input LOP3 XOR trees for free.
//  * Block-parallel kernel (CBC decrypt, ECB both ways): each warp streams a
//    contiguous range of blocks; with even blocks-per-page (the default) each
//    lane owns two consecutive blocks (1 KiB per warp step, coalesced
//    LDG.256/STG.256 -- or, for device-memory input, two texel fetches
//    through the texture pipe, off the LSU data pipe the lookups saturate),
//    else one (512 B, LDG.128).  The CBC predecessor C_{j-1}
//    comes from the neighbouring lane by one rotate-SHFL (lane 0: the previous
//    unit's lane 31, or the IV at a page start); the next unit's load is in
//    flight while the current unit's rounds run.
//  * Chain kernel (CBC encrypt, serial within a page): one thread per page
//    chain, pages balanced over a persistent grid of one CTA per SM; two
//    blocks per 256-bit L1::no_allocate load/store (measured, profiles/r1_ldst).
//  * Mixed-key kernels: same bodies; round keys of the lane's page from a
//    constant-bank copy of the key-table snapshot (block pairs: LDC, off the
//    saturated L1 data pipe) or in registers per page (CBC-encrypt chains).
//  * Launches use programmatic dependent launch: the table fill runs before
//    griddepcontrol.wait.
//  * In-place safety (out == in): CTAs own whole pages; inside a CTA every
//    warp snapshots the one predecessor block it needs from another warp
//    BEFORE the CTA-wide barrier that precedes the first store.
#include <stdint.h>
#include <stdlib.h>

#include "kg_internal.h"

namespace kg {

namespace {

constexpr int kThreads = 1024;
#ifndef KG_POOL_DIV
#define KG_POOL_DIV 16  // 1/KG_POOL_DIV of a CTA's pages form the tail-balancing pool
#endif
constexpr int kRegion = 65536;
constexpr int kSmemEnc = 2 * kRegion;                       // Te0..Te3
constexpr int kSmemDec = 2 * kRegion + 255 * 256 + 128;     // Td0..Td3 + Si (t = 0 slots only)

__device__ BaseTables g_tables;
// CBC-encrypt chain kernels: CTA page ranges start at multiples of this many
// pages.  A warp's 32 lanes walk 32 consecutive pages 4 KiB apart; with CTA
// ranges starting at an odd page or 2 mod 4 those CTAs ran 2% slower (~1,752
// vs ~1,708 us per C3 launch, bimodal by the range's start), and the launch
// waited for them: aligned to 4 pages C3 goes 604 -> 617 GB/s and the CTAs'
// finishing spread 42 -> 5 us (profiles/r2_chain_align).  KG_CHAIN_ALIGN
// overrides it (A/B).
constexpr unsigned long long kChainAlign = 4;
__constant__ unsigned long long c_chain_align = kChainAlign;
unsigned long long g_chain_align = kChainAlign;  // host copy (grid sizing)
#ifdef KG_CTA_STAMPS
// diagnostics build (tools/cta_stamps.cu): %globaltimer per CTA of the last 8
// launches: [0] start, [1] tables filled, [2] griddepcontrol.wait returned,
// [3 + w] warp w done (<= 32 warps)
constexpr int kStampW = 38;  // + [35] clock64 at the wait release, [36] clock64 at the end (thread 0), [37] %smid
__device__ unsigned long long g_stamps[8][148][kStampW];
__device__ unsigned int g_stamp_ctr;
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#endif

__device__ __forceinline__ uint32_t rotl32(uint32_t v, int s) { return __funnelshift_l(v, v, s); }

// KG_BOUNDS_CHECK (diagnostics build, `make bounds` -> build/exp/libkgpu_bounds.so;
// it stands in for compute-sanitizer memcheck, which this pool does not run):
// every global page, IV and key-id access is checked against its batch's
// extent and a violation traps (KG_ECUDA at kg_wait).  The product build
// compiles the checks away.
#ifdef KG_BOUNDS_CHECK
#define KG_CHK(c)             \
    do {                      \
        if (!(c)) __trap();   \
    } while (0)
#else
#define KG_CHK(c) \
    do {          \
    } while (0)
#endif

// Replicate the 256-entry base tables into the lane-private layout.  Warp w
// owns entries [w*per, (w+1)*per): its lanes fetch them with ONE coalesced
// load per table (all loads in flight at once), then the warp writes the 32
// lane replicas of one entry per step (entry broadcast by SHFL; lane l
// stores to bank l: conflict-free STS).  A per-thread strided loop over the
// 8192 (entry, lane) pairs instead serialised ~16 dependent global loads per
// thread (a 3.7 us prologue, profiles/r1_tail); this one is about one load
// latency plus 5*per STS per warp.
template <bool DEC>
__device__ __forceinline__ void fill_tables(char *sm) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int per = (256 + nw - 1) / nw;  // <= 32 for blockDim >= 256 (every kernel here)
    const int x0 = warp * per;
    const int xl = x0 + lane;
    const bool mine = lane < per && xl < 256;
    const uint32_t v_l = mine ? (DEC ? g_tables.td0[xl] : g_tables.te0[xl]) : 0u;
    const uint32_t s_l = (DEC && mine) ? g_tables.isb4[xl] : 0u;
#pragma unroll 4
    for (int k = 0; k < per; ++k) {
        const uint32_t v = __shfl_sync(0xffffffffu, v_l, k);
        const uint32_t sb = DEC ? __shfl_sync(0xffffffffu, s_l, k) : 0u;
        const int x = x0 + k;
        if (x < 256) {
            const int o = x * 256 + lane * 4;
            *reinterpret_cast<uint32_t *>(sm + o) = v;
            *reinterpret_cast<uint32_t *>(sm + o + 128) = rotl32(v, 8);
            *reinterpret_cast<uint32_t *>(sm + kRegion + o) = rotl32(v, 16);
            *reinterpret_cast<uint32_t *>(sm + kRegion + o + 128) = rotl32(v, 24);
            if (DEC) *reinterpret_cast<uint32_t *>(sm + 2 * kRegion + o) = sb;
        }
    }
}

// Table I (0..3) looked up with byte I of x:  T_I[x.byte(I)].
template <int I>
__device__ __forceinline__ uint32_t T(const char *sm, uint32_t x, uint32_t lb) {
    constexpr uint32_t sel = 0x7700u | (I << 4) | (4 + (I & 1));
    const uint32_t off = __byte_perm(x, lb, sel);
    return *reinterpret_cast<const uint32_t *>(sm + (I >> 1) * kRegion + off);
}

// Inverse S-box (replicated in all four bytes) looked up with byte K of x.
template <int K>
__device__ __forceinline__ uint32_t IS(const char *sm, uint32_t x, uint32_t lb) {
    constexpr uint32_t sel = 0x7700u | (K << 4) | 4;
    const uint32_t off = __byte_perm(x, lb, sel);
    return *reinterpret_cast<const uint32_t *>(sm + 2 * kRegion + off);
}

// ---- encryption: FIPS-197 §5.1 rounds in T-table form ----------------------
// Input s already XORed with round key 0 (and, for CBC, with C_{j-1}).
template <int NR>
__device__ __forceinline__ uint4 encrypt_rounds(const char *sm, uint32_t lb, uint4 s, const RoundKeys &rk) {
    uint32_t s0 = s.x, s1 = s.y, s2 = s.z, s3 = s.w;
#pragma unroll
    for (int r = 1; r < NR; ++r) {
        const uint32_t t0 = T<0>(sm, s0, lb) ^ T<1>(sm, s1, lb) ^ T<2>(sm, s2, lb) ^ T<3>(sm, s3, lb) ^ rk.w[4 * r + 0];
        const uint32_t t1 = T<0>(sm, s1, lb) ^ T<1>(sm, s2, lb) ^ T<2>(sm, s3, lb) ^ T<3>(sm, s0, lb) ^ rk.w[4 * r + 1];
        const uint32_t t2 = T<0>(sm, s2, lb) ^ T<1>(sm, s3, lb) ^ T<2>(sm, s0, lb) ^ T<3>(sm, s1, lb) ^ rk.w[4 * r + 2];
        const uint32_t t3 = T<0>(sm, s3, lb) ^ T<1>(sm, s0, lb) ^ T<2>(sm, s1, lb) ^ T<3>(sm, s2, lb) ^ rk.w[4 * r + 3];
        s0 = t0; s1 = t1; s2 = t2; s3 = t3;
    }
    // Final round (no MixColumns): S(x) is byte (I+1)%4 of T_I[x]; gather the
    // four S bytes of each column with PRMT, then AddRoundKey.
    uint4 o;
#define KG_ENC_LAST(dst, a, b, c, d, kw)                                                                  \
    dst = __byte_perm(__byte_perm(T<0>(sm, a, lb), T<1>(sm, b, lb), 0x0061u),                             \
                      __byte_perm(T<2>(sm, c, lb), T<3>(sm, d, lb), 0x4300u), 0x7610u) ^ rk.w[4 * NR + kw];
    KG_ENC_LAST(o.x, s0, s1, s2, s3, 0)
    KG_ENC_LAST(o.y, s1, s2, s3, s0, 1)
    KG_ENC_LAST(o.z, s2, s3, s0, s1, 2)
    KG_ENC_LAST(o.w, s3, s0, s1, s2, 3)
#undef KG_ENC_LAST
    return o;
}

// ---- decryption: FIPS-197 §5.3.5 equivalent inverse cipher ------------------
// Input s already XORed with dk[0] (= w[Nr]).  Returns the state after the
// final AddRoundKey (dk[Nr] = w[0]); the CBC XOR is applied by the caller.
template <int NR>
__device__ __forceinline__ uint4 decrypt_rounds(const char *sm, uint32_t lb, uint4 s, const RoundKeys &dk) {
    uint32_t s0 = s.x, s1 = s.y, s2 = s.z, s3 = s.w;
#pragma unroll
    for (int r = 1; r < NR; ++r) {
        const uint32_t t0 = T<0>(sm, s0, lb) ^ T<1>(sm, s3, lb) ^ T<2>(sm, s2, lb) ^ T<3>(sm, s1, lb) ^ dk.w[4 * r + 0];
        const uint32_t t1 = T<0>(sm, s1, lb) ^ T<1>(sm, s0, lb) ^ T<2>(sm, s3, lb) ^ T<3>(sm, s2, lb) ^ dk.w[4 * r + 1];
        const uint32_t t2 = T<0>(sm, s2, lb) ^ T<1>(sm, s1, lb) ^ T<2>(sm, s0, lb) ^ T<3>(sm, s3, lb) ^ dk.w[4 * r + 2];
        const uint32_t t3 = T<0>(sm, s3, lb) ^ T<1>(sm, s2, lb) ^ T<2>(sm, s1, lb) ^ T<3>(sm, s0, lb) ^ dk.w[4 * r + 3];
        s0 = t0; s1 = t1; s2 = t2; s3 = t3;
    }
    uint4 o;
#define KG_DEC_LAST(dst, a, b, c, d, kw)                                                                  \
    dst = __byte_perm(__byte_perm(IS<0>(sm, a, lb), IS<1>(sm, b, lb), 0x0040u),                           \
                      __byte_perm(IS<2>(sm, c, lb), IS<3>(sm, d, lb), 0x4000u), 0x7610u) ^ dk.w[4 * NR + kw];
    KG_DEC_LAST(o.x, s0, s3, s2, s1, 0)
    KG_DEC_LAST(o.y, s1, s0, s3, s2, 1)
    KG_DEC_LAST(o.z, s2, s1, s0, s3, 2)
    KG_DEC_LAST(o.w, s3, s2, s1, s0, 3)
#undef KG_DEC_LAST
    return o;
}

__device__ __forceinline__ uint4 xor4(uint4 a, uint4 b) {
    return make_uint4(a.x ^ b.x, a.y ^ b.y, a.z ^ b.z, a.w ^ b.w);
}

__device__ __forceinline__ uint4 xor4k(uint4 a, const RoundKeys &k, int r) {
    return make_uint4(a.x ^ k.w[4 * r], a.y ^ k.w[4 * r + 1], a.z ^ k.w[4 * r + 2], a.w ^ k.w[4 * r + 3]);
}

__device__ __forceinline__ uint4 shfl4(uint4 v, int src) {
    return make_uint4(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src),
                      __shfl_sync(0xffffffffu, v.z, src), __shfl_sync(0xffffffffu, v.w, src));
}

// Streaming 128-bit global access (each byte is touched exactly once).
__device__ __forceinline__ uint4 ld_stream(const uint4 *p) { return __ldcs(p); }
__device__ __forceinline__ void st_stream(uint4 *p, uint4 v) { __stcs(p, v); }

// 256-bit (two-block) global access: LDG.E.ENL2.256 / STG.E.ENL2.256 on
// sm_100.  One L1 wavefront moves two blocks.  NOALLOC: L1::no_allocate --
// measured +3.6% on the per-thread page-chain loads of the CBC-encrypt kernel
// (profiles/r1_ldst), -1.1% on the warp-coalesced decrypt loads, so the chain
// kernel uses it and the block-pair kernel does not.  Same for the stores:
// no_allocate +3.7% on CBC encrypt (568 -> 589 GB/s), -1.1% on decrypt.
template <bool NOALLOC>
__device__ __forceinline__ void ld256(const uint4 *p, uint4 &a, uint4 &b) {
    if (NOALLOC)
        asm volatile("ld.global.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
                     : "l"(p));
    else
        asm volatile("ld.global.cs.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
                     : "l"(p));
}
template <bool NOALLOC>
__device__ __forceinline__ void st256(uint4 *p, uint4 a, uint4 b) {
    if (NOALLOC)
        asm volatile("st.global.L1::no_allocate.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(a.x), "r"(a.y),
                     "r"(a.z), "r"(a.w), "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w)
                     : "memory");
    else
        asm volatile("st.global.cs.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(a.x), "r"(a.y), "r"(a.z),
                     "r"(a.w), "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w)
                     : "memory");
}

// Balanced split of [0, n) into g parts: start of part k.
__device__ __forceinline__ uint64_t part_start(uint64_t n, uint64_t g, uint64_t k) {
    const uint64_t q = n / g, r = n % g;
    return k * q + (k < r ? k : r);
}

// A warp's contiguous share [w0, w1) of the CTA range [c0, c1) (units of one
// lane item: a block or a block group).  Small ranges (at most one 32-item
// unit per warp) go out in whole units, so every active warp runs all 32
// lanes: a balanced split of, say, one 4 KiB page's 128 block pairs over 16
// warps would leave 24 of 32 lanes idle in every lookup wavefront (4x the
// LSU time of a small launch, profiles/r2_latency).  Larger ranges are split
// evenly.
__device__ __forceinline__ void small_split(uint64_t c0, uint64_t c1, uint32_t warp, uint32_t nwarps, uint64_t &w0,
                                            uint64_t &w1) {
    if (c1 - c0 <= 32ull * nwarps) {
        w0 = c0 + 32ull * warp < c1 ? c0 + 32ull * warp : c1;
        w1 = w0 + 32 < c1 ? w0 + 32 : c1;
    } else {
        w0 = c0 + part_start(c1 - c0, nwarps, warp);
        w1 = c0 + part_start(c1 - c0, nwarps, warp + 1);
    }
}

// Programmatic dependent launch (sm_90+): the table fill above does not touch
// the batch, so it may overlap the tail of the previous kernel on the stream;
// griddepcontrol.wait then blocks until that kernel has completed and its
// memory is visible.  launch_dependents lets the next launch on the stream
// start its own prologue on SMs this grid has already vacated.
__device__ __forceinline__ void pdl_prologue_done() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

__device__ __forceinline__ uint32_t lane_bytes() {
    const uint32_t l4 = (threadIdx.x & 31) * 4;
    return l4 | ((128u + l4) << 8);
}

// ---- cipher policies -----------------------------------------------------------
// first(x) = x ^ round key 0; rounds(s) = the remaining Nr rounds (through the
// final AddRoundKey).  Param*: keys by value in the kernel parameter (constant
// bank operands).  The NSK (kg_nsk.cuh) supplies shared-memory-key policies.
// lane(page) returns the per-lane key context of a block of `page` (empty
// unless keys vary per page: the mixed-key policies below).
struct NoLane {};
template <int NR>
struct ParamEnc {
    const char *sm;
    uint32_t lb;
    const RoundKeys &k;
    __device__ __forceinline__ NoLane lane(uint64_t) const { return {}; }
    __device__ __forceinline__ uint4 first(NoLane, uint4 x) const { return xor4k(x, k, 0); }
    __device__ __forceinline__ uint4 rounds(NoLane, uint4 s) const { return encrypt_rounds<NR>(sm, lb, s, k); }
};
template <int NR>
struct ParamDec {
    const char *sm;
    uint32_t lb;
    const RoundKeys &k;
    __device__ __forceinline__ NoLane lane(uint64_t) const { return {}; }
    __device__ __forceinline__ uint4 first(NoLane, uint4 x) const { return xor4k(x, k, 0); }
    __device__ __forceinline__ uint4 rounds(NoLane, uint4 s) const { return decrypt_rounds<NR>(sm, lb, s, k); }
};

// One batch (or one CTA's share of it): where the pages are.
struct Job {
    const uint4 *in;
    uint4 *out;
    const uint4 *ivs;
    uint64_t n_pages;
    uint32_t m;
    uint32_t in_place;
    unsigned long long tex = 0;  // see LaunchArgs::tex_in
    int64_t tex_off = 0;
};

// The two input blocks of pair q (blocks 2q, 2q+1): one LDG.256, or (TEX)
// two texel fetches through the texture pipe.
template <bool TEX>
__device__ __forceinline__ void ld_pair(const Job &a, uint64_t q, uint4 &x0, uint4 &x1) {
    KG_CHK(2 * q + 1 < a.n_pages * a.m);
    if (TEX) {
        const int i = (int)(a.tex_off + 2 * (int64_t)q);
        x0 = tex1Dfetch<uint4>((cudaTextureObject_t)a.tex, i);
        x1 = tex1Dfetch<uint4>((cudaTextureObject_t)a.tex, i + 1);
    } else {
        ld256<false>(a.in + 2 * q, x0, x1);
    }
}

// ---- block-parallel body: CBC decrypt, ECB decrypt, ECB encrypt ---------------
// CTA `cta` of `ncta` processes its balanced share of the batch; each warp
// streams a contiguous sub-range 32 blocks at a time.  Contains one
// __syncthreads (all threads of the CTA must call it).
template <bool DEC, bool CBC, class Cipher>
__device__ __forceinline__ void blockpar_body(const Job &a, const Cipher &cph, uint32_t cta, uint32_t ncta) {
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const uint64_t m = a.m;

    // CTA range [c0, c1) of blocks: whole pages when in place (see header).
    uint64_t c0, c1;
    if (a.in_place) {
        c0 = part_start(a.n_pages, ncta, cta) * m;
        c1 = part_start(a.n_pages, ncta, cta + 1) * m;
    } else {
        const uint64_t nb = a.n_pages * m;
        c0 = part_start(nb, ncta, cta);
        c1 = part_start(nb, ncta, cta + 1);
    }
    uint64_t w0, w1;
    small_split(c0, c1, warp, nwarps, w0, w1);

    // Per-lane position of block g = w0 + lane: page and index j in page.
    uint64_t page = (w0 + lane) / m;
    uint32_t j = (uint32_t)((w0 + lane) - page * m);

    uint4 carry = make_uint4(0, 0, 0, 0);
    if (CBC && DEC) {
        // Snapshot the predecessor of this warp's first block before anyone
        // in the CTA stores (in-place safety).
        if (w0 < w1 && (w0 % m) != 0) {
            KG_CHK(w0 - 1 < a.n_pages * m);
            carry = a.in[w0 - 1];
        }
    }
    // Software pipeline: the next unit's ciphertext is in flight while the
    // current unit's rounds run (hides the HBM latency behind the lookups).
    uint4 c_next = (w0 + lane < w1) ? ld_stream(a.in + w0 + lane) : make_uint4(0, 0, 0, 0);
    __syncthreads();

    for (uint64_t u = w0; u < w1; u += 32) {
        const uint64_t g = u + lane;
        const bool act = g < w1;
        const uint4 c = c_next;
        KG_CHK(g + 32 >= w1 || g + 32 < a.n_pages * m);
        c_next = (g + 32 < w1) ? ld_stream(a.in + g + 32) : make_uint4(0, 0, 0, 0);
        uint4 prev = make_uint4(0, 0, 0, 0);
        if (CBC && DEC) {
            // rotate by one lane: lane L gets C of lane L-1; lane 0 gets this
            // unit's lane 31, which is the next unit's lane-0 predecessor.
            const uint4 r = shfl4(c, (lane + 31) & 31);
            prev = (lane == 0) ? carry : r;
            carry = r;
            KG_CHK(!(act && j == 0) || page < a.n_pages);
            if (act && j == 0) prev = a.ivs[page];
        }
        const auto kl = cph.lane(page);
        uint4 o = cph.rounds(kl, cph.first(kl, c));
        if (CBC && DEC) o = xor4(o, prev);
        KG_CHK(!act || g < a.n_pages * m);
        if (act) st_stream(a.out + g, o);
        // advance (page, j) by 32 blocks
        j += 32;
        if (j >= m) {
            if (m >= 32) {
                j -= (uint32_t)m;
                ++page;
            } else {
                page += j / (uint32_t)m;
                j %= (uint32_t)m;
            }
        }
    }
}

// ---- block-pair body (m even): each lane owns two consecutive blocks --------
// Same contract as blockpar_body, but a warp unit is 64 blocks (1 KiB) moved
// with one LDG.256/STG.256 per lane; the CBC predecessor of the lane's first
// block is the previous lane's second block (one 4-word SHFL per 64 blocks),
// that of its second block is its own first block.  A pair never straddles a
// page (m even, ranges in whole pairs).

// G-block groups (G = 2: the block pairs above; G = 4, quads, was measured
// 10% slower -- 126 registers, profiles/r1_tex/quad -- and is not instantiated).
// A lane owns blocks G*q .. G*q+G-1 of group q; a warp unit is 32 groups.
// The CBC predecessor of the lane's first block is the previous lane's last
// block (one 4-word SHFL per unit), those of its other blocks are its own.
template <int G, bool TEX>
__device__ __forceinline__ void ld_group(const Job &a, uint64_t q, uint4 (&x)[G]) {
#pragma unroll
    for (int h = 0; h < G / 2; ++h) ld_pair<TEX>(a, (uint64_t)(G / 2) * q + h, x[2 * h], x[2 * h + 1]);
}

// Stream the groups [w0, w1) of one warp.  nx holds the warp's first unit
// (already loaded); carry = C of the block before w0 (if not a page start).
template <int G, bool DEC, bool CBC, bool TEX, class Cipher>
__device__ __forceinline__ void group_stream(const Job &a, const Cipher &cph, uint64_t w0, uint64_t w1, uint64_t mg,
                                             uint4 carry, uint64_t page, uint32_t jg, uint4 (&nx)[G]) {
    const uint32_t lane = threadIdx.x & 31;
    for (uint64_t u = w0; u < w1; u += 32) {
        const uint64_t q = u + lane;
        const bool act = q < w1;
        uint4 x[G];
#pragma unroll
        for (int b = 0; b < G; ++b) x[b] = nx[b];
        if (q + 32 < w1) ld_group<G, TEX>(a, q + 32, nx);
        uint4 prev = make_uint4(0, 0, 0, 0);
        if (CBC && DEC) {
            const uint4 r = shfl4(x[G - 1], (lane + 31) & 31);
            prev = (lane == 0) ? carry : r;
            carry = r;
            KG_CHK(!(act && jg == 0) || page < a.n_pages);
            if (act && jg == 0) prev = a.ivs[page];
        }
        const auto kl = cph.lane(page);
        uint4 o[G];
#pragma unroll
        for (int b = 0; b < G; ++b) o[b] = cph.rounds(kl, cph.first(kl, x[b]));
        if (CBC && DEC) {
            o[0] = xor4(o[0], prev);
#pragma unroll
            for (int b = 1; b < G; ++b) o[b] = xor4(o[b], x[b - 1]);
        }
        if (act) {
#pragma unroll
            for (int h = 0; h < G / 2; ++h) {
                KG_CHK(G * q + 2 * h + 1 < a.n_pages * a.m);
                st256<false>(a.out + G * q + 2 * h, o[2 * h], o[2 * h + 1]);
            }
        }
        jg += 32;
        if (jg >= mg) {
            if (mg >= 32) {
                jg -= (uint32_t)mg;
                ++page;
            } else {
                page += jg / (uint32_t)mg;
                jg %= (uint32_t)mg;
            }
        }
    }
}

// Tail balancing (large batches, pages of >= 1 KiB): the warp arbiter does not
// progress the 32 warps of a CTA evenly -- with equal static shares the last
// warp finished ~16 us (5%) after the first (profiles/r1_tail).  So only the
// first 15/16 of a CTA's pages are split statically; the rest is a pool that
// warps drain once their static share is done: 32-group units out of place
// (the unit's CBC predecessor is re-read from `in`, which nobody writes),
// whole pages in place (the IV starts each page, so no predecessor crosses
// warps).
template <int G, bool DEC, bool CBC, bool TEX, class Cipher>
__device__ __forceinline__ void blockgroup_body(const Job &a, const Cipher &cph, uint32_t cta, uint32_t ncta) {
    __shared__ unsigned long long pool_next;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const uint64_t mg = a.m / G;  // groups per page
    const bool pool = mg >= 32 && a.n_pages >= 64ull * ncta;
    uint64_t c0, c1, cmid;        // CTA range in groups; the pool is [cmid, c1)
    if (pool || a.in_place) {
        const uint64_t P0 = part_start(a.n_pages, ncta, cta), P1 = part_start(a.n_pages, ncta, cta + 1);
        c0 = P0 * mg;
        c1 = P1 * mg;
        cmid = pool ? (P1 - (P1 - P0) / KG_POOL_DIV) * mg : c1;
        if (threadIdx.x == 0) pool_next = cmid;
    } else {
        const uint64_t ng = a.n_pages * mg;
        c0 = part_start(ng, ncta, cta);
        c1 = part_start(ng, ncta, cta + 1);
        cmid = c1;
    }
    uint64_t w0, w1;
    small_split(c0, cmid, warp, nwarps, w0, w1);
    uint64_t page = (w0 + lane) / mg;
    uint32_t jg = (uint32_t)((w0 + lane) - page * mg);  // group index in the page

    uint4 carry = make_uint4(0, 0, 0, 0);
    if (CBC && DEC) {
        if (w0 < w1 && (w0 % mg) != 0) {
            KG_CHK(G * w0 - 1 < a.n_pages * a.m);
            carry = a.in[G * w0 - 1];
        }
    }
    uint4 nx[G];
#pragma unroll
    for (int b = 0; b < G; ++b) nx[b] = make_uint4(0, 0, 0, 0);
    if (w0 + lane < w1) ld_group<G, TEX>(a, w0 + lane, nx);
    __syncthreads();
    group_stream<G, DEC, CBC, TEX>(a, cph, w0, w1, mg, carry, page, jg, nx);
    if (!pool) return;
    const uint64_t unit = a.in_place ? mg : 32;  // groups per claim
    for (;;) {
        unsigned long long q0 = 0;
        if (lane == 0) q0 = atomicAdd(&pool_next, (unsigned long long)unit);
        q0 = __shfl_sync(0xffffffffu, q0, 0);
        if (q0 >= c1) break;
        // per-lane page / group index (a 32-group unit may cross a page boundary
        // when mg is not a multiple of 32)
        const uint64_t pg = (q0 + lane) / mg;
        const uint32_t jl = (uint32_t)(q0 + lane - pg * mg);
        if (q0 + lane < c1) ld_group<G, TEX>(a, q0 + lane, nx);
        uint4 cr = make_uint4(0, 0, 0, 0);
        KG_CHK(!(CBC && DEC && q0 % mg != 0) || G * q0 - 1 < a.n_pages * a.m);
        if (CBC && DEC && q0 % mg != 0) cr = a.in[G * q0 - 1];  // out of place only (in place: q0 is a page start)
        const uint64_t q1 = q0 + unit < c1 ? q0 + unit : c1;  // the last unit may be partial
        group_stream<G, DEC, CBC, TEX>(a, cph, q0, q1, mg, cr, pg, jl, nx);
    }
}

template <bool DEC, bool CBC, bool TEX = false, class Cipher>
__device__ __forceinline__ void blockpair_body(const Job &a, const Cipher &cph, uint32_t cta, uint32_t ncta) {
    blockgroup_body<2, DEC, CBC, TEX>(a, cph, cta, ncta);
}

// ---- chain body: CBC encrypt, one thread per page chain ------------------------
// WIDE (m even): blocks move two at a time with 256-bit loads/stores.
template <bool WIDE, class Cipher, bool TEX = false>
__device__ __forceinline__ void cbc_enc_body(const Job &a, const Cipher &cph, uint32_t cta, uint32_t ncta) {
    const uint32_t m = a.m;
    // CTA page ranges start at multiples of c_chain_align pages (see kChainAlign)
    const uint64_t A = c_chain_align;
    const uint64_t nu = (a.n_pages + A - 1) / A;
    uint64_t p0 = part_start(nu, ncta, cta) * A, p1 = part_start(nu, ncta, cta + 1) * A;
    if (p0 > a.n_pages) p0 = a.n_pages;
    if (p1 > a.n_pages) p1 = a.n_pages;
    for (uint64_t p = p0 + threadIdx.x; p < p1; p += blockDim.x) {
        const uint4 *src = a.in + p * m;
        uint4 *dst = a.out + p * m;
        KG_CHK(p < a.n_pages);  // the page's blocks [p*m, p*m + m) and its IV
        uint4 prev = a.ivs[p];  // C_{p,-1} := IV_p
        const auto kl = cph.lane(p);
        if (WIDE) {
            uint4 x0, x1;
            // TEX: page loads through the texture pipe (see ld_pair); pair index of block j = (p*m + j) / 2
            if (TEX) ld_pair<true>(a, (p * m) >> 1, x0, x1);
            else ld256<true>(src, x0, x1);
            for (uint32_t j = 0; j < m; j += 2) {
                uint4 n0 = x0, n1 = x1;
                if (j + 2 < m) {  // prefetch P_{j+2}, P_{j+3}
                    if (TEX) ld_pair<true>(a, (p * m + j + 2) >> 1, n0, n1);
                    else ld256<true>(src + j + 2, n0, n1);
                }
                // C_j = E_K(P_j ^ C_{j-1}); the first AddRoundKey folds into the same XOR
                const uint4 c0 = cph.rounds(kl, cph.first(kl, xor4(x0, prev)));
                prev = cph.rounds(kl, cph.first(kl, xor4(x1, c0)));
                st256<true>(dst + j, c0, prev);
                x0 = n0;
                x1 = n1;
            }
        } else {
            uint4 x = src[0];
            for (uint32_t j = 0; j < m; ++j) {
                uint4 xn = x;
                if (j + 1 < m) xn = src[j + 1];  // prefetch P_{j+1} (read before C_j is stored)
                prev = cph.rounds(kl, cph.first(kl, xor4(x, prev)));
                dst[j] = prev;
                x = xn;
            }
        }
    }
}

__device__ __forceinline__ Job job_of(const LaunchArgs &a) {
    Job j;
    j.in = a.in;
    j.out = a.out;
    j.ivs = a.ivs;
    j.n_pages = a.n_pages;
    j.m = a.m;
    j.in_place = a.in_place;
    j.tex = a.tex_in;
    j.tex_off = a.tex_off;
    return j;
}

// ---- launch-per-batch kernels -------------------------------------------------
// 512 threads + a 1/16 pool measured best (profiles/r1_tail: 256..1024 threads,
// pools of 1/4, 1/8, 1/16): 16 warps still saturate the LDS pipe and the
// 89-register budget avoids the spills of the 64-register 1024-thread build.
#ifndef KG_PAIR_TPB
#define KG_PAIR_TPB 512
#endif
constexpr int kPairThreads = KG_PAIR_TPB;  // threads per CTA of the block-pair kernels

template <int NR, int DIR, int MODE, bool PAIR, bool TEX = false>
__global__ void __launch_bounds__(PAIR ? kPairThreads : kThreads, 1) kg_blockpar(const __grid_constant__ LaunchArgs a) {
    extern __shared__ __align__(16) char sm[];
    constexpr bool DEC = (DIR == 1);
    constexpr bool CBC = (MODE == 0);
#ifdef KG_CTA_STAMPS
    const unsigned long long t_start = gtimer();
    __shared__ unsigned stamp_slot;
    if (threadIdx.x == 0) stamp_slot = (atomicAdd(&g_stamp_ctr, 1u) / gridDim.x) & 7u;
#endif
    fill_tables<DEC>(sm);
#ifdef KG_CTA_STAMPS
    __syncthreads();
    const unsigned long long t_filled = gtimer();
#endif
    pdl_prologue_done();
#ifdef KG_CTA_STAMPS
    const unsigned long long t_waited = gtimer();
    const unsigned long long c_waited = clock64();
#endif
    const uint32_t lb = lane_bytes();
    if (PAIR) {
        if (DEC) blockpair_body<true, CBC, TEX>(job_of(a), ParamDec<NR>{sm, lb, a.rk}, blockIdx.x, gridDim.x);
        else blockpair_body<false, CBC, TEX>(job_of(a), ParamEnc<NR>{sm, lb, a.rk}, blockIdx.x, gridDim.x);
    } else {
        if (DEC) blockpar_body<true, CBC>(job_of(a), ParamDec<NR>{sm, lb, a.rk}, blockIdx.x, gridDim.x);
        else blockpar_body<false, CBC>(job_of(a), ParamEnc<NR>{sm, lb, a.rk}, blockIdx.x, gridDim.x);
    }
#ifdef KG_CTA_STAMPS
    const unsigned long long t_end = gtimer();
    unsigned long long *st = g_stamps[stamp_slot][blockIdx.x];
    if ((threadIdx.x & 31) == 0) st[3 + (threadIdx.x >> 5)] = t_end;
    if (threadIdx.x == 0) {
        st[0] = t_start;
        st[1] = t_filled;
        st[2] = t_waited;
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        st[kStampW - 1] = smid;
        st[kStampW - 3] = c_waited;
        st[kStampW - 2] = clock64();
    }
#endif
}

#ifndef KG_CHAIN_TPB
#define KG_CHAIN_TPB 1024
#endif
constexpr int kChainThreads = KG_CHAIN_TPB;  // threads per CTA of the CBC-encrypt chain kernel

template <int NR, bool WIDE, bool TEX = false>
__global__ void __launch_bounds__(kChainThreads, 1) kg_cbc_enc(const __grid_constant__ LaunchArgs a) {
    extern __shared__ __align__(16) char sm[];
#ifdef KG_CTA_STAMPS
    const unsigned long long t_start = gtimer();
    __shared__ unsigned stamp_slot;
    if (threadIdx.x == 0) stamp_slot = (atomicAdd(&g_stamp_ctr, 1u) / gridDim.x) & 7u;
#endif
    fill_tables<false>(sm);
#ifdef KG_CTA_STAMPS
    __syncthreads();
    const unsigned long long t_filled = gtimer();
#endif
    pdl_prologue_done();
    __syncthreads();
#ifdef KG_CTA_STAMPS
    const unsigned long long t_waited = gtimer();
    const unsigned long long c_waited = clock64();
#endif
    cbc_enc_body<WIDE, ParamEnc<NR>, TEX>(job_of(a), ParamEnc<NR>{sm, lane_bytes(), a.rk}, blockIdx.x, gridDim.x);
#ifdef KG_CTA_STAMPS
    const unsigned long long t_end = gtimer();
    unsigned long long *st = g_stamps[stamp_slot][blockIdx.x];
    if ((threadIdx.x & 31) == 0) st[3 + (threadIdx.x >> 5)] = t_end;
    if (threadIdx.x == 0) {
        st[0] = t_start;
        st[1] = t_filled;
        st[2] = t_waited;
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        st[kStampW - 1] = smid;
        st[kStampW - 3] = c_waited;
        st[kStampW - 2] = clock64();
    }
#endif
}

// ---- mixed-key batches -------------------------------------------------------
// Round keys come from a device snapshot of the key table, per lane (the key of
// the lane's page), one 16-byte load per round; lanes of a warp usually share
// a page, so the loads broadcast.
template <int NR>
__device__ __forceinline__ uint4 keyed_encrypt_rounds(const char *sm, uint32_t lb, uint4 s, const uint4 *k) {
    uint32_t s0 = s.x, s1 = s.y, s2 = s.z, s3 = s.w;
#pragma unroll
    for (int r = 1; r < NR; ++r) {
        const uint4 kr = __ldg(k + r);
        const uint32_t t0 = T<0>(sm, s0, lb) ^ T<1>(sm, s1, lb) ^ T<2>(sm, s2, lb) ^ T<3>(sm, s3, lb) ^ kr.x;
        const uint32_t t1 = T<0>(sm, s1, lb) ^ T<1>(sm, s2, lb) ^ T<2>(sm, s3, lb) ^ T<3>(sm, s0, lb) ^ kr.y;
        const uint32_t t2 = T<0>(sm, s2, lb) ^ T<1>(sm, s3, lb) ^ T<2>(sm, s0, lb) ^ T<3>(sm, s1, lb) ^ kr.z;
        const uint32_t t3 = T<0>(sm, s3, lb) ^ T<1>(sm, s0, lb) ^ T<2>(sm, s1, lb) ^ T<3>(sm, s2, lb) ^ kr.w;
        s0 = t0; s1 = t1; s2 = t2; s3 = t3;
    }
    const uint4 kl = __ldg(k + NR);
    uint4 o;
#define KG_ENC_LAST(dst, a, b, c, d, kw)                                                                  \
    dst = __byte_perm(__byte_perm(T<0>(sm, a, lb), T<1>(sm, b, lb), 0x0061u),                             \
                      __byte_perm(T<2>(sm, c, lb), T<3>(sm, d, lb), 0x4300u), 0x7610u) ^ kw;
    KG_ENC_LAST(o.x, s0, s1, s2, s3, kl.x)
    KG_ENC_LAST(o.y, s1, s2, s3, s0, kl.y)
    KG_ENC_LAST(o.z, s2, s3, s0, s1, kl.z)
    KG_ENC_LAST(o.w, s3, s0, s1, s2, kl.w)
#undef KG_ENC_LAST
    return o;
}

template <int NR>
__device__ __forceinline__ uint4 keyed_decrypt_rounds(const char *sm, uint32_t lb, uint4 s, const uint4 *k) {
    uint32_t s0 = s.x, s1 = s.y, s2 = s.z, s3 = s.w;
#pragma unroll
    for (int r = 1; r < NR; ++r) {
        const uint4 kr = __ldg(k + r);
        const uint32_t t0 = T<0>(sm, s0, lb) ^ T<1>(sm, s3, lb) ^ T<2>(sm, s2, lb) ^ T<3>(sm, s1, lb) ^ kr.x;
        const uint32_t t1 = T<0>(sm, s1, lb) ^ T<1>(sm, s0, lb) ^ T<2>(sm, s3, lb) ^ T<3>(sm, s2, lb) ^ kr.y;
        const uint32_t t2 = T<0>(sm, s2, lb) ^ T<1>(sm, s1, lb) ^ T<2>(sm, s0, lb) ^ T<3>(sm, s3, lb) ^ kr.z;
        const uint32_t t3 = T<0>(sm, s3, lb) ^ T<1>(sm, s2, lb) ^ T<2>(sm, s1, lb) ^ T<3>(sm, s0, lb) ^ kr.w;
        s0 = t0; s1 = t1; s2 = t2; s3 = t3;
    }
    const uint4 kl = __ldg(k + NR);
    uint4 o;
#define KG_DEC_LAST(dst, a, b, c, d, kw)                                                                  \
    dst = __byte_perm(__byte_perm(IS<0>(sm, a, lb), IS<1>(sm, b, lb), 0x0040u),                           \
                      __byte_perm(IS<2>(sm, c, lb), IS<3>(sm, d, lb), 0x4000u), 0x7610u) ^ kw;
    KG_DEC_LAST(o.x, s0, s3, s2, s1, kl.x)
    KG_DEC_LAST(o.y, s1, s0, s3, s2, kl.y)
    KG_DEC_LAST(o.z, s2, s1, s0, s3, kl.z)
    KG_DEC_LAST(o.w, s3, s2, s1, s0, kl.w)
#undef KG_DEC_LAST
    return o;
}

template <int NR, bool DEC>
struct KeyedPolicy {
    const char *sm;
    uint32_t lb;
    const uint4 (*tab)[15];  // enc or dec schedules of the snapshot
    const uint8_t *nr;
    const uint16_t *ids;
    uint32_t *status;
    uint64_t n_pages;
    struct L {
        const uint4 *k;
    };
    __device__ __forceinline__ L lane(uint64_t page) const {
        if (page >= n_pages) page = n_pages - 1;  // inactive tail lanes
        uint32_t id = __ldg(ids + page);
        if (id >= (uint32_t)kMaxKeys || nr[id] != NR) {
            atomicOr(status, 1u);
            id = 0;
        }
        return L{tab[id]};
    }
    __device__ __forceinline__ uint4 first(L l, uint4 x) const { return xor4(x, __ldg(l.k)); }
    __device__ __forceinline__ uint4 rounds(L l, uint4 s) const {
        return DEC ? keyed_decrypt_rounds<NR>(sm, lb, s, l.k) : keyed_encrypt_rounds<NR>(sm, lb, s, l.k);
    }
};

// Generic round functions over a key accessor key(r) -> uint4 (round key r).
template <int NR, class KeyAt>
__device__ __forceinline__ uint4 enc_rounds_k(const char *sm, uint32_t lb, uint4 s, const KeyAt &key) {
    uint32_t s0 = s.x, s1 = s.y, s2 = s.z, s3 = s.w;
#pragma unroll
    for (int r = 1; r < NR; ++r) {
        const uint4 kr = key(r);
        const uint32_t t0 = T<0>(sm, s0, lb) ^ T<1>(sm, s1, lb) ^ T<2>(sm, s2, lb) ^ T<3>(sm, s3, lb) ^ kr.x;
        const uint32_t t1 = T<0>(sm, s1, lb) ^ T<1>(sm, s2, lb) ^ T<2>(sm, s3, lb) ^ T<3>(sm, s0, lb) ^ kr.y;
        const uint32_t t2 = T<0>(sm, s2, lb) ^ T<1>(sm, s3, lb) ^ T<2>(sm, s0, lb) ^ T<3>(sm, s1, lb) ^ kr.z;
        const uint32_t t3 = T<0>(sm, s3, lb) ^ T<1>(sm, s0, lb) ^ T<2>(sm, s1, lb) ^ T<3>(sm, s2, lb) ^ kr.w;
        s0 = t0; s1 = t1; s2 = t2; s3 = t3;
    }
    const uint4 kl = key(NR);
    uint4 o;
#define KG_ENC_LAST(dst, a, b, c, d, kw)                                                                  \
    dst = __byte_perm(__byte_perm(T<0>(sm, a, lb), T<1>(sm, b, lb), 0x0061u),                             \
                      __byte_perm(T<2>(sm, c, lb), T<3>(sm, d, lb), 0x4300u), 0x7610u) ^ kw;
    KG_ENC_LAST(o.x, s0, s1, s2, s3, kl.x)
    KG_ENC_LAST(o.y, s1, s2, s3, s0, kl.y)
    KG_ENC_LAST(o.z, s2, s3, s0, s1, kl.z)
    KG_ENC_LAST(o.w, s3, s0, s1, s2, kl.w)
#undef KG_ENC_LAST
    return o;
}

template <int NR, class KeyAt>
__device__ __forceinline__ uint4 dec_rounds_k(const char *sm, uint32_t lb, uint4 s, const KeyAt &key) {
    uint32_t s0 = s.x, s1 = s.y, s2 = s.z, s3 = s.w;
#pragma unroll
    for (int r = 1; r < NR; ++r) {
        const uint4 kr = key(r);
        const uint32_t t0 = T<0>(sm, s0, lb) ^ T<1>(sm, s3, lb) ^ T<2>(sm, s2, lb) ^ T<3>(sm, s1, lb) ^ kr.x;
        const uint32_t t1 = T<0>(sm, s1, lb) ^ T<1>(sm, s0, lb) ^ T<2>(sm, s3, lb) ^ T<3>(sm, s2, lb) ^ kr.y;
        const uint32_t t2 = T<0>(sm, s2, lb) ^ T<1>(sm, s1, lb) ^ T<2>(sm, s0, lb) ^ T<3>(sm, s3, lb) ^ kr.z;
        const uint32_t t3 = T<0>(sm, s3, lb) ^ T<1>(sm, s2, lb) ^ T<2>(sm, s1, lb) ^ T<3>(sm, s0, lb) ^ kr.w;
        s0 = t0; s1 = t1; s2 = t2; s3 = t3;
    }
    const uint4 kl = key(NR);
    uint4 o;
#define KG_DEC_LAST(dst, a, b, c, d, kw)                                                                  \
    dst = __byte_perm(__byte_perm(IS<0>(sm, a, lb), IS<1>(sm, b, lb), 0x0040u),                           \
                      __byte_perm(IS<2>(sm, c, lb), IS<3>(sm, d, lb), 0x4000u), 0x7610u) ^ kw;
    KG_DEC_LAST(o.x, s0, s3, s2, s1, kl.x)
    KG_DEC_LAST(o.y, s1, s0, s3, s2, kl.y)
    KG_DEC_LAST(o.z, s2, s1, s0, s3, kl.z)
    KG_DEC_LAST(o.w, s3, s2, s1, s0, kl.w)
#undef KG_DEC_LAST
    return o;
}

// The launch direction's schedules of a key-table snapshot in the constant
// bank (kg_load_const_keys copies them in stream order before the launch):
// a warp whose lanes share a page reads its round key with one uniform LDC
// per round from the constant cache, which does not occupy the L1 data pipe
// the table lookups saturate.
__constant__ uint4 c_keys[kMaxKeys][15];
__constant__ uint8_t c_nr[kMaxKeys];

template <int NR, bool DEC>
struct ConstKeyPolicy {
    const char *sm;
    uint32_t lb;
    const uint16_t *ids;
    uint32_t *status;
    uint64_t n_pages;
    struct L {
        uint32_t id;
    };
    struct KeyAt {
        uint32_t id;
        __device__ __forceinline__ uint4 operator()(int r) const { return c_keys[id][r]; }
    };
    __device__ __forceinline__ L lane(uint64_t page) const {
        if (page >= n_pages) page = n_pages - 1;  // inactive tail lanes
        uint32_t id = __ldg(ids + page);
        if (id >= (uint32_t)kMaxKeys || c_nr[id] != NR) {
            atomicOr(status, 1u);
            id = 0;
        }
        return L{id};
    }
    __device__ __forceinline__ uint4 first(L l, uint4 x) const { return xor4(x, c_keys[l.id][0]); }
    __device__ __forceinline__ uint4 rounds(L l, uint4 s) const {
        return DEC ? dec_rounds_k<NR>(sm, lb, s, KeyAt{l.id}) : enc_rounds_k<NR>(sm, lb, s, KeyAt{l.id});
    }
};

// Chain (CBC-encrypt) threads each own a page, so the lanes of a warp
// generally hold different keys: the page's whole schedule is loaded into
// registers once per page (Nr+1 16-byte loads per 4 KiB chain).
template <int NR>
struct RegKeyPolicy {
    const char *sm;
    uint32_t lb;
    const uint4 (*tab)[15];
    const uint8_t *nr;
    const uint16_t *ids;
    uint32_t *status;
    uint64_t n_pages;
    struct L {
        uint4 k[NR + 1];
    };
    struct KeyAt {
        const L &l;
        __device__ __forceinline__ uint4 operator()(int r) const { return l.k[r]; }
    };
    __device__ __forceinline__ L lane(uint64_t page) const {
        KG_CHK(page < n_pages);
        uint32_t id = __ldg(ids + page);
        if (id >= (uint32_t)kMaxKeys || nr[id] != NR) {
            atomicOr(status, 1u);
            id = 0;
        }
        L l;
#pragma unroll
        for (int r = 0; r <= NR; ++r) l.k[r] = __ldg(&tab[id][r]);
        return l;
    }
    __device__ __forceinline__ uint4 first(const L &l, uint4 x) const { return xor4(x, l.k[0]); }
    __device__ __forceinline__ uint4 rounds(const L &l, uint4 s) const { return enc_rounds_k<NR>(sm, lb, s, KeyAt{l}); }
};

// Mixed-key block-pair kernel (m even): CBC decrypt, ECB both ways.
// CONSTK: round keys from the constant bank (ConstKeyPolicy), else per-lane
// __ldg from the device snapshot (KeyedPolicy).
template <int NR, int DIR, int MODE, bool CONSTK, bool TEX = false>
__global__ void __launch_bounds__(kPairThreads, 1) kg_keyed_pair(const __grid_constant__ LaunchArgs a, KeyedArgs k) {
    extern __shared__ __align__(16) char sm[];
    constexpr bool DEC = (DIR == 1);
    constexpr bool CBC = (MODE == 0);
    fill_tables<DEC>(sm);
    pdl_prologue_done();
    const uint32_t lb = lane_bytes();
    if (CONSTK) {
        const ConstKeyPolicy<NR, DEC> pol{sm, lb, k.key_ids, k.status, a.n_pages};
        blockpair_body<DEC, CBC, TEX>(job_of(a), pol, blockIdx.x, gridDim.x);
    } else {
        const KeyedPolicy<NR, DEC> pol{sm, lb, DEC ? k.tab->dec : k.tab->enc, k.tab->nr, k.key_ids, k.status, a.n_pages};
        blockpair_body<DEC, CBC>(job_of(a), pol, blockIdx.x, gridDim.x);
    }
}

// Mixed-key CBC encrypt: one chain per thread, the page's keys in registers.
template <int NR, bool WIDE, bool TEX = false>
__global__ void __launch_bounds__(kPairThreads, 1) kg_keyed_chain(const __grid_constant__ LaunchArgs a, KeyedArgs k) {
    extern __shared__ __align__(16) char sm[];
    fill_tables<false>(sm);
    pdl_prologue_done();
    __syncthreads();
    const RegKeyPolicy<NR> pol{sm, lane_bytes(), k.tab->enc, k.tab->nr, k.key_ids, k.status, a.n_pages};
    cbc_enc_body<WIDE, RegKeyPolicy<NR>, TEX>(job_of(a), pol, blockIdx.x, gridDim.x);
}

template <int NR, int DIR, int MODE>
__global__ void __launch_bounds__(kThreads, 1) kg_keyed(const __grid_constant__ LaunchArgs a, KeyedArgs k) {
    extern __shared__ __align__(16) char sm[];
    constexpr bool DEC = (DIR == 1);
    constexpr bool CBC = (MODE == 0);
    fill_tables<DEC>(sm);
    pdl_prologue_done();
    const uint32_t lb = lane_bytes();
    const KeyedPolicy<NR, DEC> pol{sm, lb, DEC ? k.tab->dec : k.tab->enc, k.tab->nr, k.key_ids, k.status, a.n_pages};
    if (!DEC && CBC) {
        __syncthreads();
        cbc_enc_body<false>(job_of(a), pol, blockIdx.x, gridDim.x);
    } else {
        blockpar_body<DEC, CBC>(job_of(a), pol, blockIdx.x, gridDim.x);
    }
}

#include "kg_nsk.cuh"

template <typename K>
cudaError_t set_smem(K kernel, int bytes) {
    return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

template <int NR>
cudaError_t init_nr() {
    cudaError_t e;
    if ((e = set_smem(kg_blockpar<NR, 1, 0, false>, kSmemDec)) != cudaSuccess) return e;
    if ((e = set_smem(kg_blockpar<NR, 1, 1, false>, kSmemDec)) != cudaSuccess) return e;
    if ((e = set_smem(kg_blockpar<NR, 0, 1, false>, kSmemEnc)) != cudaSuccess) return e;
    if ((e = set_smem(kg_blockpar<NR, 1, 0, true>, kSmemDec)) != cudaSuccess) return e;
    if ((e = set_smem(kg_blockpar<NR, 1, 1, true>, kSmemDec)) != cudaSuccess) return e;
    if ((e = set_smem(kg_blockpar<NR, 0, 1, true>, kSmemEnc)) != cudaSuccess) return e;
    if ((e = set_smem(kg_blockpar<NR, 1, 0, true, true>, kSmemDec)) != cudaSuccess) return e;
    if ((e = set_smem(kg_blockpar<NR, 1, 1, true, true>, kSmemDec)) != cudaSuccess) return e;
    if ((e = set_smem(kg_blockpar<NR, 0, 1, true, true>, kSmemEnc)) != cudaSuccess) return e;
    if ((e = set_smem(kg_cbc_enc<NR, true>, kSmemEnc)) != cudaSuccess) return e;
    if ((e = set_smem(kg_cbc_enc<NR, false>, kSmemEnc)) != cudaSuccess) return e;
    if ((e = set_smem(kg_cbc_enc<NR, true, true>, kSmemEnc)) != cudaSuccess) return e;
    if ((e = set_smem(kg_keyed<NR, 1, 0>, kSmemDec)) != cudaSuccess) return e;
    if ((e = set_smem(kg_keyed<NR, 1, 1>, kSmemDec)) != cudaSuccess) return e;
    if ((e = set_smem(kg_keyed<NR, 0, 1>, kSmemEnc)) != cudaSuccess) return e;
    if ((e = set_smem(kg_keyed<NR, 0, 0>, kSmemEnc)) != cudaSuccess) return e;
    if ((e = set_smem(kg_keyed_pair<NR, 1, 0, true>, kSmemDec)) != cudaSuccess) return e;
    if ((e = set_smem(kg_keyed_pair<NR, 1, 1, true>, kSmemDec)) != cudaSuccess) return e;
    if ((e = set_smem(kg_keyed_pair<NR, 0, 1, true>, kSmemEnc)) != cudaSuccess) return e;
    if ((e = set_smem(kg_keyed_pair<NR, 1, 0, true, true>, kSmemDec)) != cudaSuccess) return e;
    if ((e = set_smem(kg_keyed_pair<NR, 1, 1, true, true>, kSmemDec)) != cudaSuccess) return e;
    if ((e = set_smem(kg_keyed_pair<NR, 0, 1, true, true>, kSmemEnc)) != cudaSuccess) return e;
    if ((e = set_smem(kg_keyed_pair<NR, 1, 0, false>, kSmemDec)) != cudaSuccess) return e;
    if ((e = set_smem(kg_keyed_pair<NR, 1, 1, false>, kSmemDec)) != cudaSuccess) return e;
    if ((e = set_smem(kg_keyed_pair<NR, 0, 1, false>, kSmemEnc)) != cudaSuccess) return e;
    if ((e = set_smem(kg_keyed_chain<NR, true>, kSmemEnc)) != cudaSuccess) return e;
    if ((e = set_smem(kg_keyed_chain<NR, false>, kSmemEnc)) != cudaSuccess) return e;
    if ((e = set_smem(kg_keyed_chain<NR, true, true>, kSmemEnc)) != cudaSuccess) return e;
    return cudaSuccess;
}

// Launch with the programmatic-stream-serialization attribute (PDL).
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl_tpb(void (*kernel)(KArgs...), unsigned grid, unsigned tpb, int smem, cudaStream_t st,
                           const Args &...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(tpb);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    static const int use_pdl = [] {
        const char *e = getenv("KG_PDL");
        return (e && *e == '0') ? 0 : 1;
    }();
    cfg.numAttrs = use_pdl;
    return cudaLaunchKernelEx(&cfg, kernel, args...);
}

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), unsigned grid, int smem, cudaStream_t st, const Args &...args) {
    return launch_pdl_tpb(kernel, grid, kThreads, smem, st, args...);
}

template <int NR>
cudaError_t launch_nr(int dir, int mode, const LaunchArgs &a, int num_sms, cudaStream_t st) {
    const uint64_t nb = a.n_pages * (uint64_t)a.m;
    if (dir == 0 && mode == 0) {
        const uint64_t units = (a.n_pages + g_chain_align - 1) / g_chain_align;  // CTA ranges of whole units
        const unsigned grid = (unsigned)(units < (uint64_t)num_sms ? units : (uint64_t)num_sms);
        const bool wide = wide_ok(a.m, a.in, a.out);
        if (wide && a.tex_in)
            return launch_pdl_tpb(kg_cbc_enc<NR, true, true>, grid, kChainThreads, kSmemEnc, st, a);
        if (wide) return launch_pdl_tpb(kg_cbc_enc<NR, true>, grid, kChainThreads, kSmemEnc, st, a);
        return launch_pdl_tpb(kg_cbc_enc<NR, false>, grid, kChainThreads, kSmemEnc, st, a);
    }
    // one CTA per 64 blocks (one warp unit of block pairs) up to one per SM:
    // small batches spread over many SMs, each filling its tables in parallel
    // (zero-copy batches: one per 256 blocks, profiles/r2_latency)
    uint64_t want = a.host_io ? (nb + 255) / 256 : (nb + 63) / 64;
    if (want > (uint64_t)num_sms) want = (uint64_t)num_sms;
    if (a.in_place && want > a.n_pages) want = a.n_pages;
    if (want < 1) want = 1;
    const unsigned grid = (unsigned)want;
    static const int pair_ok = [] {
        const char *e = getenv("KG_PAIR");
        return (e && *e == '0') ? 0 : 1;
    }();
    const bool wide = pair_ok && wide_ok(a.m, a.in, a.out);
    if (wide && a.tex_in) {
        if (dir == 1 && mode == 0) return launch_pdl_tpb(kg_blockpar<NR, 1, 0, true, true>, grid, kPairThreads, kSmemDec, st, a);
        if (dir == 1) return launch_pdl_tpb(kg_blockpar<NR, 1, 1, true, true>, grid, kPairThreads, kSmemDec, st, a);
        return launch_pdl_tpb(kg_blockpar<NR, 0, 1, true, true>, grid, kPairThreads, kSmemEnc, st, a);
    }
    if (wide) {
        if (dir == 1 && mode == 0) return launch_pdl_tpb(kg_blockpar<NR, 1, 0, true>, grid, kPairThreads, kSmemDec, st, a);
        if (dir == 1) return launch_pdl_tpb(kg_blockpar<NR, 1, 1, true>, grid, kPairThreads, kSmemDec, st, a);
        return launch_pdl_tpb(kg_blockpar<NR, 0, 1, true>, grid, kPairThreads, kSmemEnc, st, a);
    }
    if (dir == 1 && mode == 0) return launch_pdl(kg_blockpar<NR, 1, 0, false>, grid, kSmemDec, st, a);
    if (dir == 1) return launch_pdl(kg_blockpar<NR, 1, 1, false>, grid, kSmemDec, st, a);
    return launch_pdl(kg_blockpar<NR, 0, 1, false>, grid, kSmemEnc, st, a);
}

// KG_KEYED (A/B switch): 0 = one block per lane, 1024 threads, per-lane __ldg
// keys (kg_keyed); 1 = block pairs + per-lane __ldg keys; 2 (default) = block
// pairs + constant-bank keys; CBC encrypt: register keys (1, 2) or kg_keyed (0).
int keyed_variant() {
    static const int v = [] {
        const char *e = getenv("KG_KEYED");
        return (e && *e >= '0' && *e <= '2') ? *e - '0' : 2;
    }();
    return v;
}

template <int NR>
cudaError_t launch_keyed_nr(int dir, int mode, const LaunchArgs &a, const KeyedArgs &k, int num_sms, cudaStream_t st) {
    const uint64_t nb = a.n_pages * (uint64_t)a.m;
    const bool chain = (dir == 0 && mode == 0);
    uint64_t want = chain ? (a.n_pages + g_chain_align - 1) / g_chain_align : a.host_io ? (nb + 255) / 256 : (nb + 63) / 64;
    if (want > (uint64_t)num_sms) want = (uint64_t)num_sms;
    if (a.in_place && want > a.n_pages) want = a.n_pages;
    if (want < 1) want = 1;
    const unsigned grid = (unsigned)want;
    const int v = keyed_variant();
    const bool wide = wide_ok(a.m, a.in, a.out);
    if (v > 0 && chain) {
        if (wide && a.tex_in)
            return launch_pdl_tpb(kg_keyed_chain<NR, true, true>, grid, kPairThreads, kSmemEnc, st, a, k);
        if (wide) return launch_pdl_tpb(kg_keyed_chain<NR, true>, grid, kPairThreads, kSmemEnc, st, a, k);
        return launch_pdl_tpb(kg_keyed_chain<NR, false>, grid, kPairThreads, kSmemEnc, st, a, k);
    }
    if (v > 0 && wide) {
        if (v == 2 && a.tex_in) {
            if (dir == 1 && mode == 0) return launch_pdl_tpb(kg_keyed_pair<NR, 1, 0, true, true>, grid, kPairThreads, kSmemDec, st, a, k);
            if (dir == 1) return launch_pdl_tpb(kg_keyed_pair<NR, 1, 1, true, true>, grid, kPairThreads, kSmemDec, st, a, k);
            return launch_pdl_tpb(kg_keyed_pair<NR, 0, 1, true, true>, grid, kPairThreads, kSmemEnc, st, a, k);
        }
        if (v == 2) {
            if (dir == 1 && mode == 0) return launch_pdl_tpb(kg_keyed_pair<NR, 1, 0, true>, grid, kPairThreads, kSmemDec, st, a, k);
            if (dir == 1) return launch_pdl_tpb(kg_keyed_pair<NR, 1, 1, true>, grid, kPairThreads, kSmemDec, st, a, k);
            return launch_pdl_tpb(kg_keyed_pair<NR, 0, 1, true>, grid, kPairThreads, kSmemEnc, st, a, k);
        }
        if (dir == 1 && mode == 0) return launch_pdl_tpb(kg_keyed_pair<NR, 1, 0, false>, grid, kPairThreads, kSmemDec, st, a, k);
        if (dir == 1) return launch_pdl_tpb(kg_keyed_pair<NR, 1, 1, false>, grid, kPairThreads, kSmemDec, st, a, k);
        return launch_pdl_tpb(kg_keyed_pair<NR, 0, 1, false>, grid, kPairThreads, kSmemEnc, st, a, k);
    }
    if (dir == 1 && mode == 0) return launch_pdl(kg_keyed<NR, 1, 0>, grid, kSmemDec, st, a, k);
    if (dir == 1) return launch_pdl(kg_keyed<NR, 1, 1>, grid, kSmemDec, st, a, k);
    if (mode == 1) return launch_pdl(kg_keyed<NR, 0, 1>, grid, kSmemEnc, st, a, k);
    return launch_pdl(kg_keyed<NR, 0, 0>, grid, kSmemEnc, st, a, k);
}

}  // namespace

bool keyed_uses_const_keys(int dir, int mode, uint32_t m, const void *in, const void *out) {
    return keyed_variant() == 2 && !(dir == 0 && mode == 0) && wide_ok(m, in, out);
}

bool keyed_takes_tex(int dir, int mode, uint32_t m, const void *in, const void *out) {
    return wide_ok(m, in, out) && ((dir == 0 && mode == 0) ? keyed_variant() > 0 : keyed_variant() == 2);
}

cudaError_t load_const_keys(const DevKeyTable *tab, int dir, cudaStream_t st) {
    cudaError_t e = cudaMemcpyToSymbolAsync(c_keys, dir == 1 ? (const void *)tab->dec : (const void *)tab->enc,
                                            sizeof(c_keys), 0, cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return e;
    return cudaMemcpyToSymbolAsync(c_nr, tab->nr, sizeof(c_nr), 0, cudaMemcpyDeviceToDevice, st);
}

cudaError_t launch_pages_keyed(int dir, int mode, int nr, const LaunchArgs &a, const KeyedArgs &k, int num_sms,
                               cudaStream_t st) {
    switch (nr) {
        case 10: return launch_keyed_nr<10>(dir, mode, a, k, num_sms, st);
        case 12: return launch_keyed_nr<12>(dir, mode, a, k, num_sms, st);
        case 14: return launch_keyed_nr<14>(dir, mode, a, k, num_sms, st);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t kernels_init(const BaseTables &t) {
    cudaError_t e = cudaMemcpyToSymbol(g_tables, &t, sizeof(BaseTables));
    if (e != cudaSuccess) return e;
    if ((e = set_smem(kg_nsk, kSmemNsk)) != cudaSuccess) return e;
    if (const char *r = getenv("KG_CHAIN_ALIGN")) {
        const unsigned long long v = strtoull(r, nullptr, 0);
        if (v >= 1) {
            if ((e = cudaMemcpyToSymbol(c_chain_align, &v, sizeof v)) != cudaSuccess) return e;
            g_chain_align = v;
        }
    }
    if ((e = init_nr<10>()) != cudaSuccess) return e;
    if ((e = init_nr<12>()) != cudaSuccess) return e;
    return init_nr<14>();
}

cudaError_t launch_pages(int dir, int mode, int nr, const LaunchArgs &a, int num_sms, cudaStream_t st) {
    switch (nr) {
        case 10: return launch_nr<10>(dir, mode, a, num_sms, st);
        case 12: return launch_nr<12>(dir, mode, a, num_sms, st);
        case 14: return launch_nr<14>(dir, mode, a, num_sms, st);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_nsk(NskRing *ring_dev, NskCtl *ctl, uint64_t seq0, uint64_t idle_ns, int ctas, cudaStream_t st) {
    void *args[] = {&ring_dev, &ctl, &seq0, &idle_ns};
    return cudaLaunchCooperativeKernel((const void *)kg_nsk, dim3(ctas), dim3(kThreads), args, kSmemNsk, st);
}

}  // namespace kg
