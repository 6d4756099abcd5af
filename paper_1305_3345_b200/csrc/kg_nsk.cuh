// kg_nsk.cuh -- the Non-Stop Kernel (NSK): a persistent AES page service
// (row f3).  Included by kg_kernels.cu inside its anonymous namespace (it
// reuses the lookup helpers and the batch bodies there).
//
// Paper: "The NSK is small, is launched only once, and does not terminate.
// To communicate with the NSK, we have implemented a new CPU-GPU message-based
// communication method ... We use pinned memory to pass these messages"
// (PAPER.md:328-341); "When the NSK receives the message, it calls the
// service function, passing it pointers to the input buffer and output
// buffer. When the function completes, the NSK sends a completion message to
// the CPU side, and resumes polling for new request messages".
//
// B200 realisation:
//  * the request ring, doorbells and completion words live in host-mapped
//    pinned memory (NskRing); CTA 0's thread 0 polls the next doorbell over
//    the host link (ld.acquire.sys), copies the 288-byte request into device
//    memory and publishes it to every CTA through one L2 word (work_seq);
//  * every CTA then runs its balanced share of the request with the same
//    batch bodies as the launch-per-batch kernels; the last CTA to finish
//    (device-scope counter) fences at system scope and stores the sequence
//    number into the pinned completion word the host spins on;
//  * one shared-memory layout serves both directions, so the tables are
//    filled ONCE per NSK lifetime: Td0..Td3 in regions 0/1, the inverse
//    S-box in region 2's t=0 slots and Te0 in region 2's t=1 slots
//    (encryption derives Te1..Te3 by rotation: 12 extra ALU ops per
//    block-round, the price of keeping decryption at full speed);
//  * round keys change per request, so they sit in shared memory and are
//    read as one broadcast LDS.128 per round;
//  * idle watchdog: without a posted request for idle_ns (and no request
//    handed out but not yet rung -- NskRing::posted), the kernel exits after
//    a store/fence/load handshake on NskRing::exiting vs ::posted that the
//    host mirrors (so a request posted during the exit is never lost); the
//    host relaunches it on the next submit.  Process exit also ends it.

constexpr int kSmemNsk = 3 * kRegion + 16 * 16;  // tables + 15 round keys (uint4)

__device__ __forceinline__ uint64_t globaltimer_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ uint64_t ld_acquire_sys_u64(const uint64_t *p) {
    uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys_u64(uint64_t *p, uint64_t v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_sys_u64(uint64_t *p, uint64_t v) {
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void fence_sc_sys() { asm volatile("fence.sc.sys;" ::: "memory"); }
__device__ __forceinline__ unsigned long long ld_acquire_gpu_u64(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_gpu_u64(unsigned long long *p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ void fill_tables_nsk(char *sm) {
    for (int idx = threadIdx.x; idx < 256 * 32; idx += blockDim.x) {
        const int x = idx >> 5, l = idx & 31;
        const uint32_t v = g_tables.td0[x];
        const int o = x * 256 + l * 4;
        *reinterpret_cast<uint32_t *>(sm + o) = v;
        *reinterpret_cast<uint32_t *>(sm + o + 128) = rotl32(v, 8);
        *reinterpret_cast<uint32_t *>(sm + kRegion + o) = rotl32(v, 16);
        *reinterpret_cast<uint32_t *>(sm + kRegion + o + 128) = rotl32(v, 24);
        *reinterpret_cast<uint32_t *>(sm + 2 * kRegion + o) = g_tables.isb4[x];
        *reinterpret_cast<uint32_t *>(sm + 2 * kRegion + o + 128) = g_tables.te0[x];
    }
}

// Te0 (region 2, t = 1 slots) looked up with byte K of x.
template <int K>
__device__ __forceinline__ uint32_t TE0(const char *sm, uint32_t x, uint32_t lb) {
    constexpr uint32_t sel = 0x7700u | (K << 4) | 5;
    const uint32_t off = __byte_perm(x, lb, sel);
    return *reinterpret_cast<const uint32_t *>(sm + 2 * kRegion + off);
}

// Encryption with one table: T_I[x] = rotl(Te0[x], 8I).
template <int NR>
__device__ __forceinline__ uint4 nsk_encrypt_rounds(const char *sm, uint32_t lb, uint4 s, const uint4 *ks) {
    uint32_t s0 = s.x, s1 = s.y, s2 = s.z, s3 = s.w;
#pragma unroll
    for (int r = 1; r < NR; ++r) {
        const uint4 k = ks[r];
#define KG_NSK_COL(a, b, c, d, kw)                                                                       \
    (TE0<0>(sm, a, lb) ^ rotl32(TE0<1>(sm, b, lb) ^ rotl32(TE0<2>(sm, c, lb) ^ rotl32(TE0<3>(sm, d, lb), 8), 8), 8) ^ kw)
        const uint32_t t0 = KG_NSK_COL(s0, s1, s2, s3, k.x);
        const uint32_t t1 = KG_NSK_COL(s1, s2, s3, s0, k.y);
        const uint32_t t2 = KG_NSK_COL(s2, s3, s0, s1, k.z);
        const uint32_t t3 = KG_NSK_COL(s3, s0, s1, s2, k.w);
#undef KG_NSK_COL
        s0 = t0; s1 = t1; s2 = t2; s3 = t3;
    }
    // final round: S(x) is byte 1 of Te0[x]
    const uint4 k = ks[NR];
    uint4 o;
#define KG_NSK_LAST(dst, a, b, c, d, kw)                                                                  \
    dst = __byte_perm(__byte_perm(TE0<0>(sm, a, lb), TE0<1>(sm, b, lb), 0x0051u),                         \
                      __byte_perm(TE0<2>(sm, c, lb), TE0<3>(sm, d, lb), 0x5100u), 0x7610u) ^ kw;
    KG_NSK_LAST(o.x, s0, s1, s2, s3, k.x)
    KG_NSK_LAST(o.y, s1, s2, s3, s0, k.y)
    KG_NSK_LAST(o.z, s2, s3, s0, s1, k.z)
    KG_NSK_LAST(o.w, s3, s0, s1, s2, k.w)
#undef KG_NSK_LAST
    return o;
}

template <int NR>
__device__ __forceinline__ uint4 nsk_decrypt_rounds(const char *sm, uint32_t lb, uint4 s, const uint4 *ks) {
    uint32_t s0 = s.x, s1 = s.y, s2 = s.z, s3 = s.w;
#pragma unroll
    for (int r = 1; r < NR; ++r) {
        const uint4 k = ks[r];
        const uint32_t t0 = T<0>(sm, s0, lb) ^ T<1>(sm, s3, lb) ^ T<2>(sm, s2, lb) ^ T<3>(sm, s1, lb) ^ k.x;
        const uint32_t t1 = T<0>(sm, s1, lb) ^ T<1>(sm, s0, lb) ^ T<2>(sm, s3, lb) ^ T<3>(sm, s2, lb) ^ k.y;
        const uint32_t t2 = T<0>(sm, s2, lb) ^ T<1>(sm, s1, lb) ^ T<2>(sm, s0, lb) ^ T<3>(sm, s3, lb) ^ k.z;
        const uint32_t t3 = T<0>(sm, s3, lb) ^ T<1>(sm, s2, lb) ^ T<2>(sm, s1, lb) ^ T<3>(sm, s0, lb) ^ k.w;
        s0 = t0; s1 = t1; s2 = t2; s3 = t3;
    }
    const uint4 k = ks[NR];
    uint4 o;
#define KG_DEC_LAST(dst, a, b, c, d, kw)                                                                  \
    dst = __byte_perm(__byte_perm(IS<0>(sm, a, lb), IS<1>(sm, b, lb), 0x0040u),                           \
                      __byte_perm(IS<2>(sm, c, lb), IS<3>(sm, d, lb), 0x4000u), 0x7610u) ^ kw;
    KG_DEC_LAST(o.x, s0, s3, s2, s1, k.x)
    KG_DEC_LAST(o.y, s1, s0, s3, s2, k.y)
    KG_DEC_LAST(o.z, s2, s1, s0, s3, k.z)
    KG_DEC_LAST(o.w, s3, s2, s1, s0, k.w)
#undef KG_DEC_LAST
    return o;
}

template <int NR>
struct SmemEnc {
    const char *sm;
    uint32_t lb;
    const uint4 *ks;
    __device__ __forceinline__ NoLane lane(uint64_t) const { return {}; }
    __device__ __forceinline__ uint4 first(NoLane, uint4 x) const { return xor4(x, ks[0]); }
    __device__ __forceinline__ uint4 rounds(NoLane, uint4 s) const { return nsk_encrypt_rounds<NR>(sm, lb, s, ks); }
};
template <int NR>
struct SmemDec {
    const char *sm;
    uint32_t lb;
    const uint4 *ks;
    __device__ __forceinline__ NoLane lane(uint64_t) const { return {}; }
    __device__ __forceinline__ uint4 first(NoLane, uint4 x) const { return xor4(x, ks[0]); }
    __device__ __forceinline__ uint4 rounds(NoLane, uint4 s) const { return nsk_decrypt_rounds<NR>(sm, lb, s, ks); }
};

template <int NR>
__device__ __forceinline__ void nsk_run(const Job &j, uint32_t op, const char *sm, const uint4 *ks, uint32_t lb) {
    const bool dec = (op & 1) != 0, ecb = (op & 2) != 0;
    if (dec) {
        if (ecb) blockpar_body<true, false>(j, SmemDec<NR>{sm, lb, ks}, blockIdx.x, gridDim.x);
        else blockpar_body<true, true>(j, SmemDec<NR>{sm, lb, ks}, blockIdx.x, gridDim.x);
    } else if (ecb) {
        blockpar_body<false, false>(j, SmemEnc<NR>{sm, lb, ks}, blockIdx.x, gridDim.x);
    } else {
        cbc_enc_body<false>(j, SmemEnc<NR>{sm, lb, ks}, blockIdx.x, gridDim.x);
    }
}

__global__ void __launch_bounds__(kThreads, 1) kg_nsk(NskRing *ring, NskCtl *ctl, uint64_t seq0, uint64_t idle_ns) {
    extern __shared__ __align__(16) char sm[];
    uint4 *ks = reinterpret_cast<uint4 *>(sm + 3 * kRegion);
    __shared__ __align__(16) NskReq cur;
    fill_tables_nsk(sm);
    __syncthreads();
    const uint32_t lb = lane_bytes();
    for (uint64_t seq = seq0;; ++seq) {
        const int slot = (int)((seq - 1) % kNskSlots);
        if (blockIdx.x == 0 && threadIdx.x < 32) {
            // warp 0 of CTA 0: lane 0 polls the host doorbell for request `seq`,
            // then the 18 uint4 of the request cross the host link in parallel.
            int quit = 0;
            if (threadIdx.x == 0) {
                uint64_t t0 = globaltimer_ns();
                while (ld_acquire_sys_u64(&ring->doorbell[slot]) != seq) {
                    if (globaltimer_ns() - t0 > idle_ns) {
                        // Idle exit handshake with the host (Dekker): announce the
                        // exit, fence, then re-read `posted`.  The host stores
                        // `posted`, fences, then reads `exiting` (nsk_post), so at
                        // least one side sees the other's store: either this
                        // thread sees the new request and stays, or the host sees
                        // the announcement and relaunches after this grid ends.
                        st_relaxed_sys_u64(&ring->exiting, seq);
                        fence_sc_sys();
                        if (ld_acquire_sys_u64(&ring->posted) >= seq) {
                            st_relaxed_sys_u64(&ring->exiting, 0);  // handed out, doorbell pending: stay
                            fence_sc_sys();
                            t0 = globaltimer_ns();
                        } else {
                            quit = 1;
                            break;
                        }
                    }
                    __nanosleep(64);
                }
            }
            if (threadIdx.x == 0) ctl->stamp[slot][0] = globaltimer_ns();  // doorbell seen
            quit = __shfl_sync(0xffffffffu, quit, 0);
            constexpr int kWords = (int)(sizeof(NskReq) / 16);
            if (quit) {
                if (threadIdx.x == 0) ctl->req[slot].op = kNskOpQuit;
            } else if (threadIdx.x < kWords) {
                const uint4 *src = reinterpret_cast<const uint4 *>(&ring->req[slot]);
                reinterpret_cast<uint4 *>(&ctl->req[slot])[threadIdx.x] = __ldcv(src + threadIdx.x);
            }
            __threadfence();
            __syncwarp();
            if (threadIdx.x == 0) {
                ctl->stamp[slot][1] = globaltimer_ns();  // request copied to device memory
                st_release_gpu_u64(&ctl->work_seq, seq);
            }
        } else if (threadIdx.x == 0) {
            while (ld_acquire_gpu_u64(&ctl->work_seq) < seq) __nanosleep(32);
        }
        __syncthreads();
        // warp 0 pulls the request from L2 into shared memory, 16 bytes per lane
        if (threadIdx.x < (int)(sizeof(NskReq) / 16))
            reinterpret_cast<uint4 *>(&cur)[threadIdx.x] = reinterpret_cast<const uint4 *>(&ctl->req[slot])[threadIdx.x];
        __syncthreads();
        const uint32_t op = cur.op;
        if (op == kNskOpQuit) break;
        if (threadIdx.x < 15) ks[threadIdx.x] = reinterpret_cast<const uint4 *>(cur.rk)[threadIdx.x];
        Job j;
        j.in = reinterpret_cast<const uint4 *>(cur.in);
        j.out = reinterpret_cast<uint4 *>(cur.out);
        j.ivs = reinterpret_cast<const uint4 *>(cur.ivs);
        j.n_pages = cur.n_pages;
        j.m = cur.m;
        j.in_place = cur.in_place;
        const uint32_t nr = cur.nr;
        __syncthreads();  // ks ready; cur fully read into registers
        if (blockIdx.x == 0 && threadIdx.x == 0) ctl->stamp[slot][2] = globaltimer_ns();  // CTA 0 starts
        if (nr == 10) nsk_run<10>(j, op, sm, ks, lb);
        else if (nr == 12) nsk_run<12>(j, op, sm, ks, lb);
        else nsk_run<14>(j, op, sm, ks, lb);
        __syncthreads();  // this CTA's share is stored
        if (threadIdx.x == 0) {
            if (blockIdx.x == 0) ctl->stamp[slot][3] = globaltimer_ns();  // CTA 0 done
            // gpu-scope release per CTA; the single system-scope release below
            // is cumulative over everything that happened-before it.
            __threadfence();
            const unsigned prev = atomicAdd(&ctl->done_count[slot], 1u);
            if (prev == gridDim.x - 1) {
                __threadfence();  // acquire side of the counter
                ctl->stamp[slot][4] = globaltimer_ns();  // last CTA arrived
                ctl->done_count[slot] = 0;
                st_release_sys_u64(&ring->done[slot], seq);
                ctl->stamp[slot][5] = globaltimer_ns();  // completion stored
            }
        }
    }
}
