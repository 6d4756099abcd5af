// kg_internal.h -- shared between the runtime (kg_runtime.cpp) and the
// kernels (kg_kernels.cu).  Product code only; nothing here is shared with
// oracle/.
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace kg {

// Round keys as little-endian 32-bit column words: byte r of word c is
// state row r of column c (FIPS-197 §3.4 state s[r][c] = in[r + 4c]).
// Encryption: rk[4r + c] = w[4r + c] (FIPS-197 §5.2).
// Decryption: the equivalent inverse cipher's schedule in order of use
// (FIPS-197 §5.3.5): rk[0..3] = w[Nr], rk[4r..] = InvMixColumns(w[Nr-r])
// for 0 < r < Nr, rk[4Nr..] = w[0].
struct RoundKeys {
    uint32_t w[60];
};

// Everything one kernel launch needs, passed BY VALUE as the kernel
// parameter (the key words are then constant-bank operands that ptxas folds
// straight into LOP3 XORs).
struct LaunchArgs {
    const uint4 *in;      // [n_pages * m] 16-byte blocks
    uint4 *out;           // same layout; may equal in
    const uint4 *ivs;     // [n_pages] (CBC only)
    uint64_t n_pages;
    uint32_t m;           // blocks per page = page_bytes / 16
    uint32_t in_place;    // out == in
    RoundKeys rk;
    // Optional: a 1D linear texture (uint4 elements) over the input, so the
    // block-pair kernel's page loads use the TEX data pipe instead of the LSU
    // one the table lookups saturate (profiles/r1_tex).  in[i] is texel
    // tex_off + i.  0 = plain global loads.
    unsigned long long tex_in = 0;
    int64_t tex_off = 0;
    // 1: in/out/ivs are reached over the host link (zero-copy): small batches
    // then use fewer, larger CTAs (every CTA's first loads pay a link round trip)
    uint32_t host_io = 0;
};

// Base (unreplicated) lookup tables, built on the host by the GPU-path code
// (kg_tables.cpp) and copied to the device once at kg_init.
struct BaseTables {
    uint32_t te0[256];    // Te0[x] = {02}S(x) | S(x)<<8 | S(x)<<16 | {03}S(x)<<24
    uint32_t td0[256];    // Td0[x] = {0e}Si(x) | {09}Si(x)<<8 | {0d}Si(x)<<16 | {0b}Si(x)<<24
    uint32_t isb4[256];   // Si(x) * 0x01010101
};

// ---- Non-Stop Kernel (NSK, row f3) ---------------------------
// A persistent service kernel polls a request ring in host-mapped pinned
// memory ("We use pinned memory to pass these messages"),
// runs each request on all of its CTAs, and posts a completion back into the
// same pinned memory.  Layout shared by kg_runtime.cpp and kg_kernels.cu.
constexpr int kNskSlots = 64;
constexpr uint32_t kNskOpQuit = 0xFFFFu;

struct alignas(16) NskReq {  // written by the host, read by the NSK (16-byte aligned: copied as uint4)
    uint64_t in, out, ivs; // device-usable addresses (device memory or mapped pinned host memory)
    uint64_t n_pages;
    uint32_t m;            // blocks per page
    uint32_t op;           // dir | mode << 1, or kNskOpQuit
    uint32_t nr;
    uint32_t in_place;
    uint32_t rk[60];       // round keys of the request's direction (RoundKeys layout)
};

struct NskRing {                      // host-mapped pinned memory
    uint64_t doorbell[kNskSlots];     // = seq when request seq is posted (host store or cuStreamWriteValue64)
    uint64_t done[kNskSlots];         // = seq when request seq has completed (NSK store, system scope)
    uint64_t posted;                  // highest seq the host has handed out (idle watchdog guard)
    uint64_t exiting;                 // != 0: the NSK announced its idle exit while waiting for this seq
    uint64_t pad[6];
    NskReq req[kNskSlots];
};

static_assert(sizeof(NskReq) % 16 == 0, "NskReq is copied as uint4");

struct NskCtl {                       // device memory, private to the NSK
    unsigned long long work_seq;      // CTA 0 -> all CTAs: request `work_seq` is ready in req[]
    unsigned int done_count[kNskSlots];
    NskReq req[kNskSlots];            // CTA 0's copy of the host request (read from L2 by all CTAs)
    uint64_t stamp[kNskSlots][8];     // %globaltimer per request (diagnostics, KG_NSK_STAMPS=1)
};
static_assert(offsetof(NskRing, req) % 16 == 0 && offsetof(NskCtl, req) % 16 == 0, "aligned request slots");

// ---- mixed-key batches (row f1 extension) ------------------
constexpr int kMaxKeys = 256;
struct DevKeyTable {                 // a snapshot of the whole key table (device)
    uint4 enc[kMaxKeys][15];         // RoundKeys.w as uint4 per round
    uint4 dec[kMaxKeys][15];
    uint8_t nr[kMaxKeys];            // 0 = key id not set
};
struct KeyedArgs {
    const uint16_t *key_ids;         // [n_pages] key id per page (device-usable address)
    const DevKeyTable *tab;
    uint32_t *status;                // set to nonzero if a page names an unset / other-size key
};

// Block pairs move with 256-bit global loads/stores (ld/st.global.v8.u32),
// which need 32-byte alignment; kg.h promises only 16.  So the two-block
// ("wide") kernel variants run only when m is even and the pointers the
// kernel receives are 32-byte aligned; otherwise the one-block-per-lane
// variants (128-bit accesses) run.  Page offsets keep the alignment (m even:
// page_bytes is a multiple of 32), so one check per batch covers its chunks
// and texture windows.  nullptr (= a staging slot, cudaMalloc-aligned) passes.
inline bool wide_ok(uint32_t m, const void *in, const void *out) {
    return (m & 1u) == 0 && ((((uintptr_t)in) | ((uintptr_t)out)) & 31u) == 0;
}

// kg_tables.cpp
void build_base_tables(BaseTables *t);
int expand_key(const uint8_t *key, int key_bytes, RoundKeys *enc, RoundKeys *dec);  // returns Nr or -1

// kg_kernels.cu
cudaError_t kernels_init(const BaseTables &t);
// Enqueue one batch on `st`.  dir/mode/nr validated by the caller.
cudaError_t launch_pages(int dir, int mode, int nr, const LaunchArgs &a, int num_sms, cudaStream_t st);
// Mixed-key batch: page p uses key k.key_ids[p] (all of size nr).
cudaError_t launch_pages_keyed(int dir, int mode, int nr, const LaunchArgs &a, const KeyedArgs &k, int num_sms,
                               cudaStream_t st);
// True if a keyed launch of this shape reads its round keys from the
// constant-bank copy, which load_const_keys must have filled (in stream order)
// from the snapshot `tab` for direction `dir` before the launch.
bool keyed_uses_const_keys(int dir, int mode, uint32_t m, const void *in, const void *out);
cudaError_t load_const_keys(const DevKeyTable *tab, int dir, cudaStream_t st);
// True if a keyed launch of this shape has a texture-pipe input variant
// (LaunchArgs::tex_in honoured).
bool keyed_takes_tex(int dir, int mode, uint32_t m, const void *in, const void *out);
// Launch the NSK cooperatively with `ctas` CTAs; it expects request seq0 next
// and exits after idle_ns without a posted request (or on a quit request).
cudaError_t launch_nsk(NskRing *ring_dev, NskCtl *ctl, uint64_t seq0, uint64_t idle_ns, int ctas, cudaStream_t st);

}  // namespace kg
