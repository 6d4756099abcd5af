/*
 * kg.h -- C ABI of the B200-native KGPU page-crypto library (libkgpu.so).
 *
 * The one hot path of KGPU (arXiv 1305.3345) that this library implements:
 * AES encryption/decryption of batches of independent fixed-size pages,
 * offloaded from the OS to the GPU "as a service ... for the Linux crypto
 * subsystem" (§3.3), for "kernel tasks that depend on
 * per-page encryption/decryption, such as encrypted filesystems"
 * (PAPER.md:464-466).  Mode: CBC with one chain per page and a per-page IV
 * (BASELINE.json:5; the paper's own ECB, is KG_MODE_ECB).
 *
 * The call protocol follows the paper's four steps (§3.2):
 *   "requests one of the pinned-memory buffers, and fills it"  -> caller owns
 *        device or pinned-host buffers ("pinned memory
 *        for all buffers");
 *   "builds a service request"                                  -> arguments
 *        of kg_submit_pages (service = dir/mode, input/output buffers);
 *   "places the service request into request queue"             -> kg_submit_pages
 *        returns a ticket once the work is enqueued;
 *   "waits ... either by blocking ... or busy-waiting on the response
 *        queue"                                                  -> kg_wait / kg_poll.
 *
 * Conventions
 *   - Status: 0 = KG_OK, negative = error (KG_E*).  No exceptions, no
 *     longjmp, no torch types cross this boundary.
 *   - One context per process, bound to one GPU by kg_init (multi-GPU =
 *     one process per GPU).  Every call is thread-safe.
 *   - Any call other than kg_strerror/kg_launch_count before kg_init
 *     returns KG_ENOTINIT.
 *   - Argument errors are detected synchronously, before anything is
 *     enqueued; nothing is written to any caller buffer.
 *
 * Layout of a batch (all byte offsets are 64-bit):
 *   in / out : [n_pages][page_bytes] uint8, contiguous, 16-byte aligned.
 *              Page p, block j (16 bytes) lives at byte p*page_bytes + 16*j.
 *   ivs      : [n_pages][16] uint8, 16-byte aligned; page p's IV at 16*p,
 *              used raw as C_{p,-1} (SP 800-38A §6.2).  Ignored (may be NULL)
 *              for KG_MODE_ECB.
 *
 * Memory kinds: each of in, out, ivs must be device memory of the context's
 * GPU (or managed memory) or page-locked ("pinned") host memory registered
 * with CUDA.  Pageable host memory -> KG_EINVAL.  Mixed kinds are allowed.
 * Device batches run on `stream`; batches touching host memory are staged
 * through the library's device staging ring (6 slots by default: PAPER.md:437-440's
 * three buffers, plus room for the lagged D2H and back-to-back batches, profiles/r2_e2e) on internal copy/compute streams overlapped with each
 * other, joined back onto `stream`.
 */
#ifndef KG_H
#define KG_H

#include <stdint.h>

#if defined(__GNUC__)
#define KG_API __attribute__((visibility("default")))
#else
#define KG_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* Cipher direction (PAPER.md:445-447 encryption; 470-471 decryption). */
#define KG_ENCRYPT 0
#define KG_DECRYPT 1

/* Chaining mode.  CBC = NIST SP 800-38A §6.2, one chain per page
 * (BASELINE.json:5).  ECB = SP 800-38A §6.1, the paper's mode "for maximum
 * parallelism". */
#define KG_MODE_CBC 0
#define KG_MODE_ECB 1

/* Status codes. */
#define KG_OK        0
#define KG_EINVAL   -1  /* bad argument (see kg_submit_pages)                 */
#define KG_ENOKEY   -2  /* key_id has no key set                              */
#define KG_ENOTINIT -3  /* kg_init not called (or after kg_shutdown)          */
#define KG_EAGAIN   -4  /* ticket table full: wait on an older ticket first   */
#define KG_ENOMEM   -5  /* device staging allocation failed                   */
#define KG_ECUDA    -6  /* CUDA runtime/driver error; after an asynchronous   */
                        /* fault the process's context is dead (kg_shutdown) */
#define KG_ENOTSUP  -7  /* unsupported (e.g. no sm_100 device)                */
#define KG_ETICKET  -8  /* unknown, retired or already-claimed ticket         */

#define KG_MAX_KEYS 256
#define KG_MAX_INFLIGHT 65536

/* Bind this process to GPU `device`, build the device lookup tables, create
 * the internal streams.  Idempotent for the same device; a different device
 * while initialised -> KG_EINVAL.  Errors: KG_EINVAL (no such device),
 * KG_ENOTSUP (device is not compute capability 10.x), KG_ECUDA. */
KG_API int kg_init(int device);

/* Expand `key` (16, 24 or 32 bytes: AES-128/192/256, FIPS-197 §5.2
 * KeyExpansion) into encryption and equivalent-inverse-cipher decryption
 * round keys (FIPS-197 §5.3.5) and store them under key_id.  The key bytes
 * are copied; the caller may wipe its buffer on return.  Re-keying a key_id
 * never affects batches already submitted (keys are snapshotted at submit).
 * Errors: KG_ENOTINIT; KG_EINVAL (key NULL, key_bytes not 16/24/32, key_id
 * outside [0, KG_MAX_KEYS)). */
KG_API int kg_set_key(int key_id, const uint8_t *key, int key_bytes);

/* Submit one batch: `dir` (KG_ENCRYPT/KG_DECRYPT) in `mode` (KG_MODE_CBC/
 * KG_MODE_ECB) of n_pages pages of page_bytes each from `in` to `out`
 * (out == in, an exact alias, is allowed and gives the same bytes as
 * out-of-place), with page p's IV at ivs + 16p, under key `key_id`, ordered
 * after all work already enqueued on `stream` (a cudaStream_t; NULL = the
 * legacy default stream).  Work enqueued on `stream` after this call sees
 * the outputs.
 * Returns a ticket >= 0 (strictly increasing per process) or a status < 0:
 *   KG_EINVAL: dir/mode out of range; n_pages == 0; page_bytes == 0 or not a
 *     multiple of 16 (no padding); n_pages*page_bytes overflows 64 bits; a
 *     required pointer NULL or not 16-byte aligned; in/out partially
 *     overlapping; ivs overlapping out; key_id out of range; a pointer that
 *     is pageable host memory or another GPU's memory.
 *   KG_ENOKEY, KG_ENOTINIT, KG_EAGAIN, KG_ENOMEM, KG_ECUDA (launch failure).
 * Ownership: the caller owns in/out/ivs and keeps them valid and unmodified
 * until kg_wait/kg_poll reports completion; the library retains nothing
 * after completion. */
KG_API int64_t kg_submit_pages(int dir, int mode, const void *in, void *out,
                        uint64_t n_pages, uint32_t page_bytes,
                        const void *ivs, int key_id, void *stream);

/* Mixed-key batch (row f1 extension: one batch serves "a number of smaller
 * blocks of different tasks"): as kg_submit_pages, but page
 * p uses key key_ids[p] (uint16 per page, 2-byte aligned, device or pinned
 * host memory).  Every referenced key must be set and key_bytes long; the
 * key table is snapshotted at submit.  Host buffers take the same host path
 * as in kg_submit_pages (zero-copy, or the staging pipeline with each
 * chunk's launch reading its slice of key_ids).  A page naming an unset key or a key of another size makes
 * kg_wait return KG_ENOKEY (that page's output is unspecified).
 * Errors: as kg_submit_pages, plus KG_EINVAL for bad key_bytes or key_ids.
 * While the NSK runs, keyed batches are launched on the SMs it leaves free. */
KG_API int64_t kg_submit_pages_keyed(int dir, int mode, const void *in, void *out,
                                     uint64_t n_pages, uint32_t page_bytes,
                                     const void *ivs, const uint16_t *key_ids, int key_bytes,
                                     void *stream);

/* Block until the batch of `ticket` has completed; retire the ticket.
 * Returns KG_OK, KG_ECUDA (an asynchronous device fault), KG_ETICKET
 * (unknown / already retired / being waited on by another thread), KG_ENOKEY
 * (mixed-key batch naming an unset / other-size key). */
KG_API int kg_wait(int64_t ticket);

/* Non-blocking completion check (the paper's busy-wait mode).
 * Returns 1 = done, 0 = pending, < 0 = error (KG_ETICKET, KG_ECUDA).  Does not
 * retire the ticket: call kg_wait (which then returns at once) to retire. */
KG_API int kg_poll(int64_t ticket);

/* Drain all outstanding work, free the staging ring, streams, events and
 * tables, forget all keys.  KG_ENOTINIT if not initialised.
 * After an asynchronous device fault (KG_ECUDA from kg_wait/kg_poll) the
 * CUDA context of the process is unusable -- CUDA's sticky errors end only
 * with the process ("the process must be terminated and relaunched",
 * cudaErrorIllegalAddress et al.): kg_shutdown still succeeds and releases
 * the host-side state, a later kg_init returns KG_ECUDA, and a new process
 * starts cleanly (tests/test_errors_gpu.py). */
KG_API int kg_shutdown(void);

/* Static description of a status code; never NULL. */
KG_API const char *kg_strerror(int status);

/* Diagnostic environment switches (read once per process; defaults are the
 * measured best, each alternative kept for A/B runs -- DESIGN.md):
 *   KG_TEXIN=0       page loads by LDG instead of the texture pipe
 *   KG_TEX_MAX_ELEMS=n  texture window limit in texels (testing the windowed
 *                    launches of batches larger than one texture, 2^28 texels)
 *   KG_D2H_LAG=0|2|3 staged D2H not held back / only between equal chunks /
 *                    not for the last two chunks
 *   KG_RAMP_DOWN=0..3  end-ramp levels of a cold batch's staging schedule (default 3)
 *   KG_RAMP_WARM=0   treat every staged batch as cold (ramped auto chunks)
 *   KG_CHUNK_WARM=n  auto chunk bytes of warm / >= 1 GiB staged batches (default 32 MiB)
 *   KG_KEYED=0|1     mixed-key kernels: one block per lane / __ldg round keys
 *   KG_PAIR=0        one block per lane instead of block pairs
 *   KG_CHAIN_ALIGN=n CBC-encrypt CTA page ranges start at multiples of n pages (default 4)
 *   KG_PDL=0         no programmatic dependent launch
 *   KG_TRACE=1       per-chunk staging timeline on stderr at kg_wait
 *   KG_NSK_STAMPS=1  NSK per-request %globaltimer stamps;  KG_DEBUG=1 CUDA errors */

/* Staging pipeline for batches touching host memory: chunk size in bytes
 * (rounded down to whole pages, at least one page; 0 = auto: with the copy
 * engines idle at submit, ramped first/last chunks of 8 MiB -- 16 MiB for
 * CBC encryption, whose per-page chains need the longer copy to hide behind
 * -- and 32 MiB for batches of 1 GiB or more; 32 MiB without ramps when
 * earlier batches' copies are still queued) and number of device staging
 * slots (2..8).  Takes effect for
 * later submits.  Defaults: auto, 6 slots (PAPER.md:437-440's "three
 * buffers", doubled: the D2H of a chunk is held back until the next chunk's
 * H2D has landed, profiles/r1_lag, r2_e2e).  Environment overrides at kg_init:
 * KG_CHUNK_BYTES, KG_STAGING_SLOTS.  KG_EINVAL on bad values. */
KG_API int kg_set_pipeline(uint64_t chunk_bytes, int slots);

/* How batches touching pinned host memory reach the GPU (rows a3/a8 vs f4):
 *   KG_HOST_STAGED   copy engines move chunks through the device staging ring
 *                    (H2D || kernel || D2H on three streams);
 *   KG_HOST_ZEROCOPY the kernel reads and writes the caller's pinned pages
 *                    directly over the host link (no copies, one launch) --
 *                    the paper's §4 "save an extra copy" idea;
 *   KG_HOST_AUTO     zero-copy for batches of at most zc_max_bytes, staged above;
 *                    CBC encryption (serial per-page chains, 32-byte accesses)
 *                    is always staged.  Default: AUTO with zc_max_bytes = 32 MiB.
 * Takes effect for later submits.  Environment override at kg_init:
 * KG_HOST_PATH=0|1|2.  Errors: KG_ENOTINIT, KG_EINVAL (bad mode). */
#define KG_HOST_STAGED 0
#define KG_HOST_ZEROCOPY 1
#define KG_HOST_AUTO 2
KG_API int kg_set_host_path(int mode, uint64_t zc_max_bytes);

/* Non-Stop Kernel (row f3; §3.1, 403-408 §3.2).
 * kg_nsk_start launches ONE persistent service kernel on `ctas` SMs (0 ->
 * 16; at most the SM count) that keeps the AES tables resident in shared
 * memory and polls a request ring in mapped pinned host memory ("we use
 * pinned memory to pass these messages").  While it runs,
 * every kg_submit_pages is posted to it as a message instead of launching a
 * kernel; in/out/ivs may be device memory or pinned host memory (accessed
 * in place over the host link).  Completion is posted to pinned memory and
 * kg_wait busy-waits on it.
 * flags: 0 (ordered) -- the doorbell is rung by `stream` itself
 *   (cuStreamWriteValue64), so the request runs after earlier work on
 *   `stream`, and later work on `stream` waits for it (cuStreamWaitValue64);
 *   KG_NSK_DIRECT -- the host rings the doorbell at submit (lowest latency;
 *   ordering with `stream` is then the caller's job).
 * idle_ms: the kernel exits after this long without requests (0 -> 2000 ms)
 * and is relaunched transparently by the next submit.  The NSK occupies its
 * SMs; other kernels share the remaining ones.
 * Errors: KG_ENOTINIT; KG_EINVAL (bad ctas/flags, already running);
 * KG_ENOTSUP (stream memory operations unavailable, ordered mode);
 * KG_ENOMEM; KG_ECUDA.  kg_nsk_stop drains and stops it (KG_OK if not
 * running); kg_shutdown stops it too. */
#define KG_NSK_DIRECT 1
#define KG_NSK_NOCAL 2  /* skip the start-up calibration: every request goes to the NSK */
KG_API int kg_nsk_start(int ctas, int flags, uint32_t idle_ms);
KG_API int kg_nsk_stop(void);

/* Size-based dispatch while the NSK runs (row f2; the paper's "dynamically
 * dispatching tasks ... depending on their size ... calibrate it using
 * microbenchmarks at boot time").  The library has no CPU
 * path (no CPU fallback by design), so the two legs are its two GPU paths:
 * requests of at most max_bytes (n_pages*page_bytes) go to the NSK (the
 * low-overhead path for small requests), larger ones are launched as
 * ordinary kernels on the SMs the NSK leaves free (the paper's "switches to a
 * traditional CUDA kernel launch").
 * kg_nsk_start calibrates at start unless KG_NSK_NOCAL is given: it times
 * both paths, caller-observed, on AES-128-CBC decrypt batches of 1, 2, 4, ...
 * 4 KiB pages in device memory (median of 5 after 2 warm-ups, stopping two
 * sizes after the launch first wins) and sets the threshold with
 * kg_dispatch_threshold.  max_bytes = 0 re-calibrates; UINT64_MAX sends
 * everything to the NSK; any other value is used as given.  *chosen (may be
 * NULL) receives the threshold.  Errors: KG_ENOTINIT, KG_EINVAL (NSK not
 * running), KG_ENOMEM, KG_ECUDA. */
KG_API int kg_nsk_dispatch(uint64_t max_bytes, uint64_t *chosen);

/* One calibration sample: batch size and the two paths' median latencies. */
typedef struct {
    uint64_t bytes;
    double nsk_us;
    double launch_us;
} kg_calib_point;

/* The dispatch rule (pure; no device needed): given samples sorted by size,
 * the threshold is the size of the last sample before the first one where
 * the launch is strictly faster (a tie goes to the NSK, the small-request
 * path, SPEC.md:414's tie rule); 0 if the launch wins at the first sample;
 * UINT64_MAX if it never wins (or n <= 0).  Dispatch is then monotone by
 * construction: NSK for sizes <= threshold, launches above. */
KG_API uint64_t kg_dispatch_threshold(const kg_calib_point *pts, int n);

/* Copy up to max_pts samples of the last calibration into pts; returns the
 * number of samples it has (0 if none yet).  Errors: KG_ENOTINIT, KG_EINVAL. */
KG_API int kg_nsk_calibration(kg_calib_point *pts, int max_pts);

/* Pinned host allocations for batches (row f4; "allocate memory in the pinned
 * region ... to save an extra copy"): pinned and mapped
 * memory allocated from a thread bound to the CPUs local to the context's GPU
 * (sysfs local_cpulist), so the pages land on the GPU's NUMA node without
 * libnuma (cudaHostAlloc; KG_PINNED_MODE=register instead first-touches an
 * mmap region on those CPUs and registers it).  Usable as in/out/ivs of
 * kg_submit_pages (staged or zero-copy).  NULL if not initialised or on failure.
 * kg_free_pinned: KG_EINVAL if `p` did not come from kg_alloc_pinned. */
KG_API void *kg_alloc_pinned(uint64_t bytes);
KG_API int kg_free_pinned(void *p);

/* Number of CUDA kernels this library has launched in this process
 * (instrumentation for benchmarks; monotonic, never reset). */
KG_API uint64_t kg_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* KG_H */
