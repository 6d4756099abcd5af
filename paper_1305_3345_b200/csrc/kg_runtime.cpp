// kg_runtime.cpp -- the C ABI (include/kg.h): context, key table, request
// validation, tickets (the paper's request/response queues), and the
// pinned-host staging pipeline.
//
// Paper mapping (§3.2):
//  * "builds a service request ... places the service request into request
//    queue" -> kg_submit_pages validates, snapshots the round keys and
//    enqueues device work; the returned ticket is the queue entry.
//  * "waits ... by blocking ... or busy-waiting on the response queue"
//    -> kg_wait (cudaEventSynchronize) / kg_poll (cudaEventQuery).
//  * "the helper DMAs the input data buffer to the GPU ... This can proceed
//    concurrently with another service running on the GPU" and "on the GPU,
//    we use three buffers ... one is used by the active service, a second
//    may receive input ... a third may be copying the output" -> host-memory
//    batches stream through a ring of device staging slots (default 3) on an
//    H2D stream, a compute stream and a D2H stream ordered by events.
//  * There is no user-space helper process and no kernel module: one address
//    space, so the copy engines DMA straight from/to the caller's pinned
//    pages (the paper's own §4 "save an extra copy" idea).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <atomic>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "../../include/kg.h"
#include "kg_internal.h"

namespace {

struct KeySlot {
    bool set = false;
    int nr = 0;
    kg::RoundKeys enc, dec;
};

struct Ticket {
    cudaEvent_t ev = nullptr;
    bool claimed = false;
};

struct Slot {
    uint8_t *data = nullptr;   // chunk_pages * page_bytes
    uint8_t *ivs = nullptr;    // chunk_pages * 16
    cudaEvent_t loaded = nullptr, done = nullptr, freed = nullptr;
};

constexpr int kMaxSlots = 8;

struct Ctx {
    bool up = false;
    int device = -1;
    int num_sms = 0;
    KeySlot keys[KG_MAX_KEYS];
    int64_t next_ticket = 0;
    std::unordered_map<int64_t, Ticket> tickets;
    std::vector<cudaEvent_t> ev_pool;
    cudaStream_t s_h2d = nullptr, s_comp = nullptr, s_d2h = nullptr;
    cudaEvent_t ev_begin = nullptr;
    Slot slots[kMaxSlots];
    uint64_t chunk_bytes = 16ull << 20;
    int n_slots = 3;
    uint64_t slot_bytes = 0;   // current allocation per slot (data)
    uint64_t slot_ivs = 0;     // current allocation per slot (ivs)
    int host_path = KG_HOST_STAGED;
    uint64_t zc_max_bytes = 1ull << 20;
};

std::mutex g_mu;
Ctx g;

// KG_TRACE=1: record a timing event after every staging stage of the next
// host batch and print the per-chunk timeline (JSON, stderr) at its kg_wait.
struct TraceEv {
    uint64_t chunk;
    char stage;  // 'b' begin, 'h' H2D done, 'k' kernel done, 'd' D2H done
    cudaEvent_t ev;
};
std::vector<TraceEv> g_trace;
bool trace_on() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("KG_TRACE");
        v = (e && *e && *e != '0') ? 1 : 0;
    }
    return v == 1;
}
void trace(uint64_t chunk, char stage, cudaStream_t st) {
    if (!trace_on()) return;
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return;
    cudaEventRecord(e, st);
    g_trace.push_back({chunk, stage, e});
}
void trace_dump() {
    if (g_trace.empty()) return;
    cudaEventSynchronize(g_trace.back().ev);
    fprintf(stderr, "{\"kg_trace\": [");
    for (size_t i = 0; i < g_trace.size(); i++) {
        float ms = 0.f;
        cudaEventSynchronize(g_trace[i].ev);
        cudaEventElapsedTime(&ms, g_trace[0].ev, g_trace[i].ev);
        fprintf(stderr, "%s[%llu, \"%c\", %.2f]", i ? ", " : "", (unsigned long long)g_trace[i].chunk,
                g_trace[i].stage, ms * 1000.f);
    }
    fprintf(stderr, "]}\n");
    for (auto &t : g_trace) cudaEventDestroy(t.ev);
    g_trace.clear();
}
std::atomic<uint64_t> g_launches{0};

bool debug_on() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("KG_DEBUG");
        v = (e && *e && *e != '0') ? 1 : 0;
    }
    return v == 1;
}

int cuda_fail(cudaError_t e, const char *where) {
    if (debug_on()) fprintf(stderr, "[kg] %s: %s\n", where, cudaGetErrorString(e));
    return KG_ECUDA;
}

#define KG_CU(call)                                                  \
    do {                                                             \
        cudaError_t _e = (call);                                     \
        if (_e != cudaSuccess) return cuda_fail(_e, #call);          \
    } while (0)

cudaEvent_t take_event() {
    if (!g.ev_pool.empty()) {
        cudaEvent_t e = g.ev_pool.back();
        g.ev_pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return nullptr;
    return e;
}

void free_staging() {
    for (int i = 0; i < kMaxSlots; i++) {
        if (g.slots[i].data) cudaFree(g.slots[i].data);
        if (g.slots[i].ivs) cudaFree(g.slots[i].ivs);
        g.slots[i].data = nullptr;
        g.slots[i].ivs = nullptr;
    }
    g.slot_bytes = g.slot_ivs = 0;
}

// Make sure every slot holds at least `bytes` of data and `ivb` of IVs.
int ensure_staging(uint64_t bytes, uint64_t ivb) {
    if (g.slot_bytes >= bytes && g.slot_ivs >= ivb && g.slots[g.n_slots - 1].data) return KG_OK;
    // Growing: all staging users must be finished first.
    cudaStreamSynchronize(g.s_h2d);
    cudaStreamSynchronize(g.s_comp);
    cudaStreamSynchronize(g.s_d2h);
    uint64_t nb = bytes > g.slot_bytes ? bytes : g.slot_bytes;
    uint64_t ni = ivb > g.slot_ivs ? ivb : g.slot_ivs;
    free_staging();
    for (int i = 0; i < kMaxSlots && i < g.n_slots; i++) {
        if (cudaMalloc(&g.slots[i].data, nb) != cudaSuccess || cudaMalloc(&g.slots[i].ivs, ni) != cudaSuccess) {
            cudaGetLastError();
            free_staging();
            return KG_ENOMEM;
        }
    }
    g.slot_bytes = nb;
    g.slot_ivs = ni;
    return KG_OK;
}

enum Kind { K_BAD = 0, K_DEVICE = 1, K_HOST = 2 };

// Classify a caller pointer; for pinned host memory also return the address
// a kernel may use to reach it over the host link (UVA: usually identical).
Kind classify(const void *p, const void **dev_alias = nullptr) {
    cudaPointerAttributes at;
    cudaError_t e = cudaPointerGetAttributes(&at, p);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return K_BAD;
    }
    switch (at.type) {
        case cudaMemoryTypeDevice:
            return at.device == g.device ? K_DEVICE : K_BAD;
        case cudaMemoryTypeManaged:
            return K_DEVICE;
        case cudaMemoryTypeHost:
            if (dev_alias) {
                // devicePointer is the mapping of the allocation's base address
                *dev_alias = at.devicePointer
                                 ? (const void *)((const uint8_t *)at.devicePointer +
                                                  ((const uint8_t *)p - (const uint8_t *)at.hostPointer))
                                 : nullptr;
            }
            return K_HOST;
        default:
            return K_BAD;  // unregistered (pageable) host memory
    }
}

bool overlap(uintptr_t a, uint64_t na, uintptr_t b, uint64_t nb) { return a < b + nb && b < a + na; }

int64_t new_ticket(cudaStream_t st) {
    if (g.tickets.size() >= (size_t)KG_MAX_INFLIGHT) return KG_EAGAIN;
    cudaEvent_t ev = take_event();
    if (!ev) return KG_ECUDA;
    cudaError_t e = cudaEventRecord(ev, st);
    if (e != cudaSuccess) {
        g.ev_pool.push_back(ev);
        return cuda_fail(e, "cudaEventRecord(ticket)");
    }
    int64_t t = g.next_ticket++;
    g.tickets[t] = Ticket{ev, false};
    return t;
}

int launch(int dir, int mode, int nr, const kg::LaunchArgs &a, cudaStream_t st) {
    cudaError_t e = kg::launch_pages(dir, mode, nr, a, g.num_sms, st);
    if (e != cudaSuccess) return cuda_fail(e, "launch_pages");
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return KG_OK;
}

// Host-memory batch: chunked H2D -> compute -> D2H through the staging ring.
int submit_staged(int dir, int mode, int nr, const kg::RoundKeys &rk, const uint8_t *in, Kind kin,
                  uint8_t *out, Kind kout, uint64_t n_pages, uint32_t page_bytes, const uint8_t *ivs,
                  Kind kiv, cudaStream_t st) {
    uint64_t chunk_pages = g.chunk_bytes / page_bytes;
    if (chunk_pages < 1) chunk_pages = 1;
    if (chunk_pages > n_pages) chunk_pages = n_pages;
    const bool need_iv = (mode == KG_MODE_CBC);
    int rc = ensure_staging(chunk_pages * page_bytes, need_iv ? chunk_pages * 16 : 16);
    if (rc != KG_OK) return rc;

    KG_CU(cudaEventRecord(g.ev_begin, st));
    trace(0, 'b', st);
    KG_CU(cudaStreamWaitEvent(g.s_h2d, g.ev_begin, 0));
    KG_CU(cudaStreamWaitEvent(g.s_comp, g.ev_begin, 0));
    KG_CU(cudaStreamWaitEvent(g.s_d2h, g.ev_begin, 0));

    uint64_t i = 0;
    for (uint64_t p0 = 0; p0 < n_pages; p0 += chunk_pages, ++i) {
        const uint64_t np = (n_pages - p0 < chunk_pages) ? (n_pages - p0) : chunk_pages;
        const uint64_t off = p0 * page_bytes, nbytes = np * page_bytes;
        Slot &s = g.slots[i % (uint64_t)g.n_slots];
        // H2D stage: wait until the slot's previous output has drained.
        KG_CU(cudaStreamWaitEvent(g.s_h2d, s.freed, 0));
        if (kin == K_HOST) KG_CU(cudaMemcpyAsync(s.data, in + off, nbytes, cudaMemcpyHostToDevice, g.s_h2d));
        if (need_iv && kiv == K_HOST)
            KG_CU(cudaMemcpyAsync(s.ivs, ivs + 16 * p0, 16 * np, cudaMemcpyHostToDevice, g.s_h2d));
        KG_CU(cudaEventRecord(s.loaded, g.s_h2d));
        trace(i, 'h', g.s_h2d);
        // compute stage
        KG_CU(cudaStreamWaitEvent(g.s_comp, s.loaded, 0));
        kg::LaunchArgs a;
        a.in = reinterpret_cast<const uint4 *>(kin == K_HOST ? s.data : in + off);
        a.out = reinterpret_cast<uint4 *>(kout == K_HOST ? s.data : out + off);
        a.ivs = need_iv ? reinterpret_cast<const uint4 *>(kiv == K_HOST ? s.ivs : ivs + 16 * p0) : nullptr;
        a.n_pages = np;
        a.m = page_bytes / 16;
        a.in_place = (const void *)a.in == (const void *)a.out;
        a.rk = rk;
        rc = launch(dir, mode, nr, a, g.s_comp);
        if (rc != KG_OK) return rc;
        KG_CU(cudaEventRecord(s.done, g.s_comp));
        trace(i, 'k', g.s_comp);
        // D2H stage
        KG_CU(cudaStreamWaitEvent(g.s_d2h, s.done, 0));
        if (kout == K_HOST) KG_CU(cudaMemcpyAsync(out + off, s.data, nbytes, cudaMemcpyDeviceToHost, g.s_d2h));
        KG_CU(cudaEventRecord(s.freed, g.s_d2h));
        trace(i, 'd', g.s_d2h);
    }
    // join: the caller's stream continues after the last D2H
    KG_CU(cudaEventRecord(g.ev_begin, g.s_d2h));
    KG_CU(cudaStreamWaitEvent(st, g.ev_begin, 0));
    return KG_OK;
}

}  // namespace

extern "C" {

const char *kg_strerror(int status) {
    switch (status) {
        case KG_OK: return "ok";
        case KG_EINVAL: return "invalid argument";
        case KG_ENOKEY: return "no key set for key_id";
        case KG_ENOTINIT: return "library not initialised (kg_init)";
        case KG_EAGAIN: return "ticket table full";
        case KG_ENOMEM: return "device staging allocation failed";
        case KG_ECUDA: return "CUDA error";
        case KG_ENOTSUP: return "not supported";
        case KG_ETICKET: return "unknown or retired ticket";
        default: return status > 0 ? "pending" : "unknown status";
    }
}

uint64_t kg_launch_count(void) { return g_launches.load(); }

int kg_init(int device) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (g.up) return device == g.device ? KG_OK : KG_EINVAL;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return KG_ENOTSUP;
    }
    if (device < 0 || device >= n) return KG_EINVAL;
    KG_CU(cudaSetDevice(device));
    cudaDeviceProp prop;
    KG_CU(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) return KG_ENOTSUP;  // built for sm_100a only
    g.device = device;
    g.num_sms = prop.multiProcessorCount;
    kg::BaseTables t;
    kg::build_base_tables(&t);
    KG_CU(kg::kernels_init(t));
    KG_CU(cudaStreamCreateWithFlags(&g.s_h2d, cudaStreamNonBlocking));
    KG_CU(cudaStreamCreateWithFlags(&g.s_comp, cudaStreamNonBlocking));
    KG_CU(cudaStreamCreateWithFlags(&g.s_d2h, cudaStreamNonBlocking));
    KG_CU(cudaEventCreateWithFlags(&g.ev_begin, cudaEventDisableTiming));
    for (int i = 0; i < kMaxSlots; i++) {
        KG_CU(cudaEventCreateWithFlags(&g.slots[i].loaded, cudaEventDisableTiming));
        KG_CU(cudaEventCreateWithFlags(&g.slots[i].done, cudaEventDisableTiming));
        KG_CU(cudaEventCreateWithFlags(&g.slots[i].freed, cudaEventDisableTiming));
    }
    if (const char *e = getenv("KG_CHUNK_BYTES")) {
        unsigned long long v = strtoull(e, nullptr, 0);
        if (v >= 16) g.chunk_bytes = v;
    }
    if (const char *e = getenv("KG_HOST_PATH")) {
        int v = atoi(e);
        if (v >= KG_HOST_STAGED && v <= KG_HOST_AUTO) g.host_path = v;
    }
    if (const char *e = getenv("KG_STAGING_SLOTS")) {
        int v = atoi(e);
        if (v >= 2 && v <= kMaxSlots) g.n_slots = v;
    }
    g.up = true;
    return KG_OK;
}

int kg_set_pipeline(uint64_t chunk_bytes, int slots) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!g.up) return KG_ENOTINIT;
    if (chunk_bytes < 16 || slots < 2 || slots > kMaxSlots) return KG_EINVAL;
    if (slots != g.n_slots) {
        cudaStreamSynchronize(g.s_h2d);
        cudaStreamSynchronize(g.s_comp);
        cudaStreamSynchronize(g.s_d2h);
        free_staging();
        g.n_slots = slots;
    }
    g.chunk_bytes = chunk_bytes;
    return KG_OK;
}

int kg_set_host_path(int mode, uint64_t zc_max_bytes) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!g.up) return KG_ENOTINIT;
    if (mode != KG_HOST_STAGED && mode != KG_HOST_ZEROCOPY && mode != KG_HOST_AUTO) return KG_EINVAL;
    g.host_path = mode;
    g.zc_max_bytes = zc_max_bytes;
    return KG_OK;
}

int kg_set_key(int key_id, const uint8_t *key, int key_bytes) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!g.up) return KG_ENOTINIT;
    if (key_id < 0 || key_id >= KG_MAX_KEYS || !key) return KG_EINVAL;
    if (key_bytes != 16 && key_bytes != 24 && key_bytes != 32) return KG_EINVAL;
    KeySlot ks;
    ks.nr = kg::expand_key(key, key_bytes, &ks.enc, &ks.dec);
    if (ks.nr < 0) return KG_EINVAL;
    ks.set = true;
    g.keys[key_id] = ks;
    return KG_OK;
}

int64_t kg_submit_pages(int dir, int mode, const void *in, void *out, uint64_t n_pages, uint32_t page_bytes,
                        const void *ivs, int key_id, void *stream) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!g.up) return KG_ENOTINIT;
    if ((dir != KG_ENCRYPT && dir != KG_DECRYPT) || (mode != KG_MODE_CBC && mode != KG_MODE_ECB)) return KG_EINVAL;
    if (n_pages == 0 || page_bytes == 0 || page_bytes % 16 != 0) return KG_EINVAL;
    if (n_pages > UINT64_MAX / page_bytes) return KG_EINVAL;
    const uint64_t total = n_pages * page_bytes;
    const bool need_iv = (mode == KG_MODE_CBC);
    if (!in || !out || (need_iv && !ivs)) return KG_EINVAL;
    if (((uintptr_t)in | (uintptr_t)out) & 15u) return KG_EINVAL;
    if (need_iv && ((uintptr_t)ivs & 15u)) return KG_EINVAL;
    if (need_iv && n_pages > UINT64_MAX / 16) return KG_EINVAL;
    if (in != out && overlap((uintptr_t)in, total, (uintptr_t)out, total)) return KG_EINVAL;
    if (need_iv && overlap((uintptr_t)ivs, 16 * n_pages, (uintptr_t)out, total)) return KG_EINVAL;
    if (key_id < 0 || key_id >= KG_MAX_KEYS) return KG_EINVAL;
    const KeySlot &ks = g.keys[key_id];
    if (!ks.set) return KG_ENOKEY;
    const void *zin = in, *zout = out, *ziv = ivs;
    const Kind kin = classify(in, &zin), kout = classify(out, &zout),
               kiv = need_iv ? classify(ivs, &ziv) : K_DEVICE;
    if (kin == K_BAD || kout == K_BAD || kiv == K_BAD) return KG_EINVAL;
    if (g.tickets.size() >= (size_t)KG_MAX_INFLIGHT) return KG_EAGAIN;

    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const kg::RoundKeys &rk = (dir == KG_ENCRYPT) ? ks.enc : ks.dec;  // snapshot: copied into LaunchArgs
    int rc;
    const bool all_device = (kin == K_DEVICE && kout == K_DEVICE && kiv == K_DEVICE);
    // Zero-copy (row f4): the kernel reads and writes the
    // caller's pinned pages over the host link, no staging copies.
    const bool zero_copy = !all_device && zin && zout && (!need_iv || ziv) &&
                           (g.host_path == KG_HOST_ZEROCOPY ||
                            (g.host_path == KG_HOST_AUTO && total <= g.zc_max_bytes));
    if (all_device || zero_copy) {
        kg::LaunchArgs a;
        a.in = reinterpret_cast<const uint4 *>(zin);
        a.out = reinterpret_cast<uint4 *>(const_cast<void *>(zout));
        a.ivs = need_iv ? reinterpret_cast<const uint4 *>(ziv) : nullptr;
        a.n_pages = n_pages;
        a.m = page_bytes / 16;
        a.in_place = (in == out);
        a.rk = rk;
        rc = launch(dir, mode, ks.nr, a, st);
    } else {
        rc = submit_staged(dir, mode, ks.nr, rk, (const uint8_t *)in, kin, (uint8_t *)out, kout, n_pages,
                           page_bytes, (const uint8_t *)ivs, kiv, st);
    }
    if (rc != KG_OK) return rc;
    return new_ticket(st);
}

int kg_wait(int64_t ticket) {
    cudaEvent_t ev;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        if (!g.up) return KG_ENOTINIT;
        auto it = g.tickets.find(ticket);
        if (it == g.tickets.end() || it->second.claimed) return KG_ETICKET;
        it->second.claimed = true;
        ev = it->second.ev;
    }
    cudaError_t e = cudaEventSynchronize(ev);
    std::lock_guard<std::mutex> lk(g_mu);
    if (trace_on()) trace_dump();
    g.tickets.erase(ticket);
    g.ev_pool.push_back(ev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaEventSynchronize");
    return KG_OK;
}

int kg_poll(int64_t ticket) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!g.up) return KG_ENOTINIT;
    auto it = g.tickets.find(ticket);
    if (it == g.tickets.end() || it->second.claimed) return KG_ETICKET;
    cudaError_t e = cudaEventQuery(it->second.ev);
    if (e == cudaSuccess) return 1;
    if (e == cudaErrorNotReady) {
        cudaGetLastError();
        return 0;
    }
    return cuda_fail(e, "cudaEventQuery");
}

int kg_shutdown(void) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!g.up) return KG_ENOTINIT;
    cudaDeviceSynchronize();
    for (auto &kv : g.tickets) cudaEventDestroy(kv.second.ev);
    g.tickets.clear();
    for (cudaEvent_t e : g.ev_pool) cudaEventDestroy(e);
    g.ev_pool.clear();
    free_staging();
    for (int i = 0; i < kMaxSlots; i++) {
        cudaEventDestroy(g.slots[i].loaded);
        cudaEventDestroy(g.slots[i].done);
        cudaEventDestroy(g.slots[i].freed);
        g.slots[i].loaded = g.slots[i].done = g.slots[i].freed = nullptr;
    }
    cudaEventDestroy(g.ev_begin);
    cudaStreamDestroy(g.s_h2d);
    cudaStreamDestroy(g.s_comp);
    cudaStreamDestroy(g.s_d2h);
    g.ev_begin = nullptr;
    g.s_h2d = g.s_comp = g.s_d2h = nullptr;
    for (auto &k : g.keys) k = KeySlot();
    g.up = false;
    g.device = -1;
    cudaGetLastError();
    return KG_OK;
}

}  // extern "C"
