#!/usr/bin/env python
"""bench.py -- AES-CBC page-crypto throughput on B200 (BASELINE.json metric:
"AES-CBC page crypto GB/s (HBM & pinned-host) at 1/2/4/8 B200; % of roofline").

Headline (`value`, the configuration BASELINE.json's metric is quoted on,
configs[1] = C2): "eCryptfs-shaped read": AES-128-CBC DECRYPT of a 256 MiB
batch of 65,536 independent 4 KiB pages with per-page IVs, HBM-resident,
per GPU (weak scaling).  One step = one pass of the whole hot path over one
batch: kg_submit_pages (validate, snapshot key, enqueue) -> the decrypt
kernel -> completion ticket (kg_wait).  Keys are expanded once (kg_set_key),
outside the timed region ("key expansion once per key", BASELINE.json:5).

The same JSON line carries, under "configs", every other BASELINE config
timed the same way with its own roofline, traffic, check, e2e and clocks:
  c3       AES-256-CBC encrypt, 1 GiB per GPU (configs[2]; the north star's
           "1 GiB batches")
  c4_1gib  AES-128-CBC decrypt, 1 GiB per GPU (the top of the configs[3] sweep)
  c5       AES-128-CBC decrypt of 64 GiB in place, page-range sharded over the
           ranks (configs[4]; strong scaling: the 1/2/4/8 curve)
and "c4_sweep" (rank 0, one GPU): caller-observed latency from 1 page to
1 GiB, HBM and pinned host, beside the oracle (1 and T threads) and
single-core OpenSSL (context), with the GPU/CPU crossovers.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c2|c3|c4_1gib|c5|...]
      N > 1 without WORLD_SIZE in the environment: re-launches itself under
      torch.distributed.run with N ranks (one per GPU, NCCL).
  torchrun --nproc-per-node N ... bench.py --gpus N    (the same, launched by the caller)
  python bench.py --impl reference   (the oracle on the host cores: a bounded
                                      sample of the same workload)

Prints ONE JSON line on rank 0.  `value` = payload GB/s (10^9 page bytes per
second, IVs excluded) over all ranks, device-timed with CUDA events on the
launching stream, max over ranks.  `e2e` = the same metric through the C ABI
with NUMA-local pinned HOST buffers (H2D + kernel + D2H inside the timed
region: the pinned-host-resident figure of the metric).  DESIGN.md §9.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402

METRIC = "AES-CBC page crypto GB/s (HBM & pinned-host) at 1/2/4/8 B200; % of roofline"
PB = 4096
M_PERIOD = 65537        # C5: page p holds page p mod M of a seeded M-page set

# name: (n_pages per rank (weak) or in total (strong), key_bytes, dir, mode, in_place, scaling, description)
WORKLOADS = {
    "c2": (65536, 16, 1, 0, False, "weak",
           "C2 eCryptfs-shaped read: AES-128-CBC decrypt, 65,536 x 4 KiB pages (256 MiB) per GPU, HBM-resident, out-of-place"),
    "c3": (262144, 32, 0, 0, False, "weak",
           "C3 eCryptfs-shaped write: AES-256-CBC encrypt (page-parallel chains), 262,144 x 4 KiB pages (1 GiB) per GPU, HBM-resident"),
    "c4_1gib": (262144, 16, 1, 0, False, "weak",
                "C4 at 1 GiB (top of the batch-size sweep): AES-128-CBC decrypt, 262,144 x 4 KiB pages per GPU, HBM-resident"),
    "c5": (16777216, 16, 1, 0, True, "strong",
           "C5: AES-128-CBC decrypt of 64 GiB (16,777,216 x 4 KiB pages) page-range sharded over the ranks, HBM-resident, in place"),
    # not BASELINE configs: the paper's own ECB mode (row f1), mixed-key batches, in place
    "ecb_dec": (65536, 16, 1, 1, False, "weak", "AES-128-ECB decrypt (the paper's mode, PAPER.md:448-450), 65,536 x 4 KiB pages, HBM"),
    "ecb_enc": (65536, 16, 0, 1, False, "weak", "AES-128-ECB encrypt (the paper's mode, PAPER.md:448-450), 65,536 x 4 KiB pages, HBM"),
    "c2_keyed": (65536, 16, 1, 0, False, "weak", "C2 with a key id per page (8 AES-128 keys, uniform), HBM, out-of-place"),
    "c3_keyed": (262144, 32, 0, 0, False, "weak", "C3 with a key id per page (8 AES-256 keys, uniform), HBM, out-of-place"),
    "c2_inplace": (65536, 16, 1, 0, True, "weak", "C2 in place (AES-128-CBC decrypt, 65,536 x 4 KiB pages), HBM"),
    "ecb_dec_inplace": (65536, 16, 1, 1, True, "weak", "AES-128-ECB decrypt in place, 65,536 x 4 KiB pages, HBM"),
}
KEYED = ("c2_keyed", "c3_keyed")
DEFAULT_EXTRA = ("c3", "c4_1gib", "c5")
SM_COUNT = 148
LDS_LANES_PER_CLK = 32      # lane-lookups/clk/SM (B300_MICROARCH.md "smem crossbar 128/N B/cyc/SM"; tools/pipes.cu measures it)


def nr_of(key_bytes):
    return {16: 10, 24: 12, 32: 14}[key_bytes]


def compute_peak_gbs(key_bytes, sm_mhz, sms=SM_COUNT):
    """T-table compute ceiling in payload GB/s: 16*Nr lane-lookups per 16-byte
    block at LDS_LANES_PER_CLK per SM per clock."""
    return sms * sm_mhz * 1e6 * LDS_LANES_PER_CLK * 16.0 / (16.0 * nr_of(key_bytes)) / 1e9


# ----------------------------------------------------------------------------- multi-rank plan (tested on CPU)
def plan(workload, rank, world):
    """This rank's share of a workload: (first_page, n_pages, scaling).
    Weak scaling: every rank its own full batch (pages [rank*n, (rank+1)*n) of
    the seeded stream).  Strong scaling (C5): contiguous page range
    [floor(rN/W), floor((r+1)N/W)) of the one job."""
    n_total, _, _, _, _, scaling, _ = WORKLOADS[workload]
    if scaling == "strong":
        lo, hi = synth.shard(n_total, rank, world)
        return lo, hi - lo, scaling
    return rank * n_total, n_total, scaling


def job_bytes(workload, world, steps):
    """Payload bytes the whole job (all ranks) processes in `steps` steps."""
    n_total, _, _, _, _, scaling, _ = WORKLOADS[workload]
    per_step = n_total * PB * (world if scaling == "weak" else 1)
    return per_step * steps


def reduce_max(dist, values, device):
    """MAX over ranks of a list of floats (the timing reduction)."""
    if dist is None:
        return [float(v) for v in values]
    import torch
    t = torch.tensor([float(v) for v in values], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(v) for v in t.tolist()]


def reduce_sum(dist, values, device):
    """SUM over ranks of a list of floats (check counters)."""
    if dist is None:
        return [float(v) for v in values]
    import torch
    t = torch.tensor([float(v) for v in values], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return [float(v) for v in t.tolist()]


# ----------------------------------------------------------------------------- peaks, traffic, clocks
def load_peaks():
    """Driver-written measured peaks; tolerant of the key names (the HBM copy
    bandwidth and the max SM clock are all bench.py reads), else the
    profiling guide's fallback."""
    fallback = {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "_fallback": True}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            raw = json.load(f)
    except (OSError, ValueError):
        return fallback

    def find(pred):
        stack = [raw]
        while stack:
            x = stack.pop()
            if isinstance(x, dict):
                for k, v in x.items():
                    if isinstance(v, (int, float)) and pred(k.lower()):
                        return float(v)
                    if isinstance(v, (dict, list)):
                        stack.append(v)
            elif isinstance(x, list):
                stack.extend(x)
        return None

    hbm = find(lambda k: "hbm" in k and ("gbs" in k or "gb_s" in k or "bw" in k or "bandwidth" in k))
    mhz = find(lambda k: "max" in k and "mhz" in k)
    if hbm is None:
        return fallback
    return {"hbm_gbs": hbm, "sm_max_mhz": mhz or 1965.0, "_raw_keys": sorted(raw) if isinstance(raw, dict) else None}


def load_traffic(workload):
    """ncu dram bytes per launch for the dominant kernel, committed under profiles/."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f).get(workload)
    except (OSError, ValueError):
        return None


class ClockSampler:
    """pynvml sampling of SM clock + throttle reasons during a timed region
    (every `period` s, plus one sample at entry and one at exit)."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, pci=None, index=0, period=0.001):
        self.ok = False
        self.samples, self.reasons = [], set()
        self.period = period
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = None
            if pci is not None:  # (domain, bus, device) of the CUDA device: NVML ignores CUDA_VISIBLE_DEVICES
                for i in range(pynvml.nvmlDeviceGetCount()):
                    h = pynvml.nvmlDeviceGetHandleByIndex(i)
                    p = pynvml.nvmlDeviceGetPciInfo(h)
                    if (p.domain, p.bus, p.device) == tuple(pci):
                        self.h = h
                        break
            if self.h is None:
                self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:  # noqa: BLE001
            self.max_mhz = None
        self._stop = threading.Event()
        self._t = None

    def _one(self):
        try:
            self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
            r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            for bit, name in self.REASONS.items():
                if r & bit and bit != 0x1:
                    self.reasons.add(name)
        except Exception:  # noqa: BLE001
            pass

    def _run(self):
        while not self._stop.is_set():
            self._one()
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self._one()
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()
            self._one()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_min_mhz": min(self.samples),
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}


def merge_clocks(parts):
    """Clock summaries of several ranks / regions -> one (min of medians, union of reasons)."""
    parts = [p for p in parts if p and p.get("samples")]
    if not parts:
        return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
    return {"sm_mhz": min(p["sm_mhz"] for p in parts), "sm_min_mhz": min(p.get("sm_min_mhz", p["sm_mhz"]) for p in parts),
            "sm_max_mhz": max((p["sm_max_mhz"] or 0) for p in parts) or None,
            "reasons": sorted(set().union(*[set(p["reasons"]) for p in parts])),
            "samples": sum(p["samples"] for p in parts), "ranks_or_regions": len(parts)}


def duplex_link(torch, dist, red_dev, h_a, h_b, nbytes=128 << 20, reps=5):
    """Pinned-host link bound: concurrent H2D + D2H copies (every payload byte
    crosses the link both ways), all ranks copying at once (a barrier before
    each rep).  Returns (per-rank GB/s per direction, aggregate GB/s per
    direction over all ranks = W * bytes / max-rank time)."""
    nbytes = min(nbytes, h_a.numel(), h_b.numel())
    d_a = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    d_b = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    best, best_max = None, None
    world = dist.get_world_size() if dist else 1
    for _ in range(reps):
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        s1.wait_event(e0)
        s2.wait_event(e0)
        with torch.cuda.stream(s1):
            d_a.copy_(h_a[:nbytes], non_blocking=True)
        with torch.cuda.stream(s2):
            h_b[:nbytes].copy_(d_b, non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 1e3
        tmax = reduce_max(dist, [t], red_dev)[0]
        best = t if best is None else min(best, t)
        best_max = tmax if best_max is None else min(best_max, tmax)
    del d_a, d_b
    return nbytes / best / 1e9, world * nbytes / best_max / 1e9


# ----------------------------------------------------------------------------- oracle (reference arm / cpu_baseline)
def oracle_rate(n_pages_cap, key_bytes, direction, target_s, threads):
    """Time the oracle, as it stands, on a bounded sample of the workload.
    Returns (GB/s, pages, seconds)."""
    import oracle
    key = synth.make_key(key_bytes)
    cal = max(threads, 8)
    data = synth.make_pages(cal, PB)
    ivs = synth.make_ivs(cal)
    t0 = time.perf_counter()
    oracle.pages(direction, 0, key, data, cal, PB, ivs, threads=threads)
    rate = cal / max(time.perf_counter() - t0, 1e-6)           # pages/s
    n = int(min(n_pages_cap, max(threads, rate * target_s)))
    data = synth.make_pages(n, PB)
    ivs = synth.make_ivs(n)
    t0 = time.perf_counter()
    oracle.pages(direction, 0, key, data, n, PB, ivs, threads=threads)
    dt = time.perf_counter() - t0
    return n * PB / dt / 1e9, n, dt


def openssl_rate(key_bytes, direction, target_s=2.0):
    """Context, NOT the oracle: single-core OpenSSL (AES-NI) CBC through the
    `cryptography` package, one cipher context per 4 KiB page (as a
    filesystem would call it), on a bounded sample.  The paper's comparator
    was an SSE-optimised in-kernel AES."""
    try:
        from cryptography.hazmat.primitives.ciphers import Cipher, algorithms, modes
    except Exception as e:  # noqa: BLE001
        return {"unavailable": repr(e)}
    key = synth.make_key(key_bytes)
    n = 4096
    data = synth.make_pages(n, PB).tobytes()
    ivs = synth.make_ivs(n).tobytes()

    def one_pass():
        for p in range(n):
            c = Cipher(algorithms.AES(key), modes.CBC(ivs[16 * p:16 * p + 16]))
            x = c.decryptor() if direction else c.encryptor()
            x.update(data[p * PB:(p + 1) * PB])

    t0 = time.perf_counter()
    reps = 0
    while time.perf_counter() - t0 < target_s or reps == 0:
        one_pass()
        reps += 1
    dt = time.perf_counter() - t0
    return {"value": reps * n * PB / dt / 1e9, "unit": "GB/s", "cores": 1, "kind": "openssl_aesni_context (not the oracle)",
            "sample": f"{reps} x {n} seeded 4 KiB pages, one cipher context per page, {dt:.1f} s"}


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    n_pages, key_bytes, direction, mode, _, scaling, desc = WORKLOADS[args.workload]
    threads = len(os.sched_getaffinity(0))
    per_step = args.ref_step_seconds or max(0.5, min(10.0, 150.0 / max(1, args.steps + args.warmup)))
    import oracle
    key = synth.make_key(key_bytes)
    # calibrate the per-step sample
    _, n, dt = oracle_rate(n_pages, key_bytes, direction, per_step, threads)
    data = synth.make_pages(n, PB)
    ivs = synth.make_ivs(n)
    for _ in range(args.warmup):
        oracle.pages(direction, mode, key, data, n, PB, ivs, threads=threads)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.pages(direction, mode, key, data, n, PB, ivs, threads=threads)
        times.append(time.perf_counter() - t0)
    total = sum(times)
    gbs = n * PB * args.steps / total / 1e9
    sample = f"{n} of the workload's {n_pages} 4 KiB pages per step ({n * PB / 2**20:.1f} MiB), {threads} pthreads"
    line = {
        "impl": "reference", "metric": METRIC, "value": gbs, "unit": "GB/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": desc, "n_pages": n_pages, "page_bytes": PB, "key_bits": 8 * key_bytes,
                   "dir": "decrypt" if direction else "encrypt", "sampled_pages_per_step": n,
                   "world_ranks_present": world},
        "cpu_baseline": {"value": gbs, "unit": "GB/s", "cores": threads, "kind": "oracle", "sample": sample},
        "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- our arm
class Ctx:
    """Per-process state of our arm (rank, device, process group)."""

    def __init__(self, args):
        import torch
        self.torch = torch
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        # one process per GPU; KG_BENCH_SHARE_GPU=1 (testing the N>1 code path
        # on a one-GPU box) maps ranks onto the available devices and uses gloo
        self.share = os.environ.get("KG_BENCH_SHARE_GPU") == "1"
        self.dev = self.local % torch.cuda.device_count() if self.share else self.local
        torch.cuda.set_device(self.dev)
        self.dist = None
        self.red_dev = "cpu"
        self.comm = {"backend": None, "world": 1}
        if self.world > 1:
            import torch.distributed as dist
            if self.share:
                dist.init_process_group("gloo")
            else:
                # the NCCL log then shows the communicator's rank count (INIT lines only)
                os.environ.setdefault("NCCL_DEBUG", "INFO")
                os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
                dist.init_process_group("nccl", device_id=torch.device("cuda", self.dev))
                self.red_dev = "cuda"
            self.dist = dist
            one = torch.ones(1, dtype=torch.float64, device=self.red_dev)
            dist.all_reduce(one)
            self.comm = {"backend": dist.get_backend(), "world": dist.get_world_size(),
                         "allreduce_sum_of_ones": int(one.item())}
        try:
            pr = torch.cuda.get_device_properties(self.dev)
            self.pci = (int(pr.pci_domain_id), int(pr.pci_bus_id), int(pr.pci_device_id))
        except Exception:  # noqa: BLE001
            self.pci = None

    def barrier(self):
        self.torch.cuda.synchronize()
        if self.dist:
            self.dist.barrier()
        self.torch.cuda.synchronize()

    def gather(self, obj):
        if not self.dist:
            return [obj]
        out = [None] * self.world
        self.dist.all_gather_object(out, obj)
        return out


def make_inputs(ctx, workload, first, n):
    """Seeded device inputs of this rank (untimed).  C5: the periodic M-page pattern."""
    torch = ctx.torch
    if workload == "c5":
        M = M_PERIOD
        pat = torch.from_numpy(synth.make_pages(M, PB)).cuda().view(M, PB)
        ivp = torch.from_numpy(synth.make_ivs(M)).cuda().view(M, 16)
        x = torch.empty((n, PB), dtype=torch.uint8, device="cuda")
        ivs = torch.empty((n, 16), dtype=torch.uint8, device="cuda")
        fill_periodic(torch, x, ivs, pat, ivp, first)
        return x.view(-1), ivs.view(-1), (pat, ivp)
    x = torch.from_numpy(synth.make_pages(n, PB, first_page=first)).cuda()
    ivs = torch.from_numpy(synth.make_ivs(n, first_page=first)).cuda()
    return x, ivs, None


def fill_periodic(torch, x, ivs, pat, ivp, first):
    """x[p] = pat[(first + p) mod M] (device copies)."""
    n, M = x.shape[0], pat.shape[0]
    p = 0
    while p < n:
        src = (first + p) % M
        cnt = min(n - p, M - src)
        x[p:p + cnt].copy_(pat[src:src + cnt])
        ivs[p:p + cnt].copy_(ivp[src:src + cnt])
        p += cnt


def run_config(ctx, args, workload, steps, warmup, want_e2e=True):
    """Time one workload on every rank; returns the rank-0 summary dict (None elsewhere)."""
    import paper_1305_3345_b200 as kg
    torch = ctx.torch
    n_total, key_bytes, direction, mode, in_place, scaling, desc = WORKLOADS[workload]
    first, n, _ = plan(workload, ctx.rank, ctx.world)
    keyed = workload in KEYED
    key = synth.make_key(key_bytes)
    kg.set_key(0, key)
    if keyed:
        for i in range(8):
            kg.set_key(i, synth.make_key(key_bytes, seed=synth.KEY_SEED + 100 + i))
    stream = torch.cuda.current_stream()
    x, ivs, pattern = make_inputs(ctx, workload, first, n)
    out = x if in_place else torch.empty_like(x)
    key_ids = None
    if keyed:
        key_ids = torch.from_numpy((synth.stream_bytes(synth.KEY_SEED + 7, 2 * n).view(np.uint16) % 8)
                                   .astype(np.int16)).cuda()
    torch.cuda.synchronize()

    def step(dst=None, src=None, d=direction):
        s_in = x if src is None else src
        s_out = out if dst is None else dst
        if keyed:
            return kg.submit_pages_keyed(d, mode, s_in, s_out, n, PB, ivs if mode == 0 else None, key_ids, key_bytes,
                                         stream)
        return kg.submit_pages(d, mode, s_in, s_out, n, PB, ivs if mode == 0 else None, 0, stream)

    for _ in range(warmup):
        kg.wait(step())
    ctx.barrier()

    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(ctx.pci, ctx.dev) as clk:
        t_wall0 = time.perf_counter()
        # Q untimed steps between the barrier and the start event keep the GPU
        # busy into the timed region: the device-timed region then starts with
        # steps queued and the SMs at their steady-state speed, instead of idling
        # through Python's first submit and re-warming for ~2 ms after the
        # barrier's idle (profiles/r2_timing).  The region holds exactly K steps;
        # the host-inclusive figure is `e2e`.
        ahead = [step() for _ in range(args.queue_ahead_steps)]
        l0 = kg.launch_count()
        ev0.record(stream)
        tickets = [step() for _ in range(steps)]
        ev1.record(stream)
        for t in ahead:
            kg.wait(t)
        for t in tickets:
            kg.wait(t)
        torch.cuda.synchronize()
        t_wall = time.perf_counter() - t_wall0
    launches = kg.launch_count() - l0
    elapsed = ev0.elapsed_time(ev1) / 1e3                 # s, device-timed on the launching stream
    avg_launch = elapsed / max(launches, steps)           # launches back to back on one stream
    elapsed_max, avg_launch_max = reduce_max(ctx.dist, [elapsed, avg_launch], ctx.red_dev)
    value = job_bytes(workload, ctx.world, steps) / elapsed_max / 1e9
    clocks = merge_clocks(ctx.gather(clk.summary()))
    launches_all = int(reduce_sum(ctx.dist, [launches], ctx.red_dev)[0])

    # correctness check outside the timed region (every rank, SUM over ranks)
    check = None
    if not args.no_check:
        if workload == "c5":
            # one step on freshly filled pages; EVERY byte is compared on the
            # device with one launch over the M-page pattern (pages are
            # independent; tests/test_fullsize_gpu.py anchors that run to the oracle)
            pat, ivp = pattern
            fill_periodic(torch, x.view(n, PB), ivs.view(n, 16), pat, ivp, first)
            kg.wait(step())
            ref = torch.empty_like(pat)
            kg.wait(kg.submit_pages(direction, mode, pat, ref, M_PERIOD, PB, ivp, 0, stream))
            bad = 0
            xv = x.view(n, PB)
            for s in range(0, n, M_PERIOD):
                e = min(n, s + M_PERIOD)
                src = (first + s) % M_PERIOD
                cnt = e - s
                if src + cnt <= M_PERIOD:
                    exp = ref[src:src + cnt]
                else:
                    exp = torch.cat([ref[src:], ref[:cnt - (M_PERIOD - src)]])
                bad += int((xv[s:e] != exp).any(dim=1).sum())
            del ref
            tot = reduce_sum(ctx.dist, [bad, n], ctx.red_dev)
            check = {"pages": int(tot[1]), "mismatched_pages": int(tot[0]),
                     "method": "every byte of one fresh step vs one launch over the M=65,537-page pattern "
                               "(periodic input; oracle anchoring of that run: tests/test_fullsize_gpu.py)"}
        else:
            # one more step, then EVERY output page goes back through the
            # inverse operation on the GPU and must reproduce the step's input
            before = x.clone() if in_place else x
            kg.wait(step())
            back = torch.empty_like(x)
            inv = 1 - direction
            if keyed:
                kg.wait(kg.submit_pages_keyed(inv, mode, out, back, n, PB, ivs if mode == 0 else None, key_ids,
                                              key_bytes, stream))
            else:
                kg.wait(kg.submit_pages(inv, mode, out, back, n, PB, ivs if mode == 0 else None, 0, stream))
            torch.cuda.synchronize()
            bad = int((back.view(n, PB) != before.view(n, PB)).any(dim=1).sum())
            del back, before
            tot = reduce_sum(ctx.dist, [bad, n], ctx.red_dev)
            check = {"pages": int(tot[1]), "mismatched_pages": int(tot[0]),
                     "method": "one extra step; every output page through the inverse operation on the GPU must "
                               "give back the step's input page (byte-exact parity vs the oracle: tests/)"}
    del pattern

    # e2e through the C ABI with NUMA-local pinned HOST buffers (H2D + compute + D2H timed)
    e2e = None
    if want_e2e and not args.no_e2e and not keyed:
        big = workload == "c5"
        # C5 (64 GiB per step): 2 warm-up + 4 timed steps (~8.5 s); its first
        # steps after the buffer's allocation run slower (profiles/r2_e2e, c5_steps)
        e_steps = max(1, min(steps, 4 if big else args.e2e_steps))
        hx = kg.alloc_pinned(n * PB)
        hx.copy_(x)
        hiv = kg.alloc_pinned(16 * n)
        hiv.copy_(ivs)
        # Requests in flight: like the paper's pipelined service calls (one
        # buffer in service while the next is copied in and the previous out,
        # PAPER.md:437-440), the caller keeps `depth` batches submitted and
        # waits for the oldest; each batch in flight has its own output buffer
        # (nothing is shared between batches in flight).  In place (C5) the
        # next batch's input is the previous one's output: one at a time.
        depth = 1 if in_place else max(1, args.e2e_depth)
        houts = [hx] if in_place else [kg.alloc_pinned(n * PB) for _ in range(depth)]
        del x, out, ivs
        torch.cuda.empty_cache()
        residency = ("pinned host (kg_alloc_pinned: cudaHostAlloc from a thread on the GPU-local CPUs)"
                     + (", in place" if in_place else f", {depth} batches in flight, one output buffer each"))

        # each batch in flight on its own stream: a batch is ordered after the
        # work already on its stream (kg.h), so one stream would serialise them
        e_streams = [stream] + [torch.cuda.Stream() for _ in range(depth - 1)]

        def submit_e2e(i):
            return kg.submit_pages(direction, mode, hx, houts[i % depth], n, PB, hiv if mode == 0 else None, 0,
                                   e_streams[i % depth])

        for i in range(2):
            kg.wait(submit_e2e(i))
        ctx.barrier()
        step_ms = []
        t0 = time.perf_counter()
        inflight = []
        t_prev = t0
        for i in range(e_steps):
            if len(inflight) == depth:
                kg.wait(inflight.pop(0))
                t_now = time.perf_counter()
                step_ms.append((t_now - t_prev) * 1e3)
                t_prev = t_now
            inflight.append(submit_e2e(i))
        for t in inflight:
            kg.wait(t)
            t_now = time.perf_counter()
            step_ms.append((t_now - t_prev) * 1e3)
            t_prev = t_now
        te = time.perf_counter() - t0
        te_max = reduce_max(ctx.dist, [te], ctx.red_dev)[0]
        e2e = {"value": job_bytes(workload, ctx.world, e_steps) / te_max / 1e9, "unit": "GB/s",
               "h2d_bytes_per_step": n * PB + (16 * n if mode == 0 else 0), "d2h_bytes_per_step": n * PB,
               "steps": e_steps, "residency": residency, "batches_in_flight": depth,
               "timing": "wall clock from the first submit to the last kg_wait, max over ranks; step_ms = intervals "
                         "between successive completions",
               "step_ms_min_median_max": [round(min(step_ms), 3), round(sorted(step_ms)[len(step_ms) // 2], 3),
                                          round(max(step_ms), 3)]}
        if len(step_ms) <= 8:
            e2e["step_ms"] = [round(x, 3) for x in step_ms]
        per_rank, agg = duplex_link(torch, ctx.dist, ctx.red_dev, hx, houts[0])
        e2e["link_duplex_gbs_per_direction"] = per_rank
        e2e["link_duplex_aggregate_gbs_per_direction"] = agg
        e2e["link_frac"] = e2e["value"] / agg if agg else None
        e2e["link_note"] = ("bound = concurrent pinned H2D + D2H copies measured with all ranks copying at once "
                            "(aggregate over ranks, per direction)")
        kg.free_pinned(hx)
        kg.free_pinned(hiv)
        if not in_place:
            for h in houts:
                kg.free_pinned(h)
        del hx, houts, hiv
    else:
        del x, out, ivs
    del key_ids
    torch.cuda.empty_cache()

    if ctx.rank != 0:
        return None
    peaks = load_peaks()
    sm_max = float(clocks.get("sm_max_mhz") or peaks.get("sm_max_mhz", 1965.0))
    launches_per_step = max(1, launches // steps)
    bytes_launch = n * PB / launches_per_step
    achieved = bytes_launch / avg_launch_max / 1e9
    peak = compute_peak_gbs(key_bytes, sm_max)
    chain = direction == 0 and mode == 0
    kernel = (("kg_keyed_chain" if chain else "kg_keyed_pair") if keyed
              else "kg_cbc_enc" if chain else "kg_blockpar") + \
        f"<Nr={nr_of(key_bytes)},{'dec' if direction else 'enc'},{'ecb' if mode else 'cbc'}>"
    roof = {
        "bound": "alu", "pipe": "lds (shared-memory T-table lookups: 16*Nr lane-lookups per 16-byte block)",
        "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
        "traffic": load_traffic(workload),
        "traffic_unit": "DRAM bytes per launch (ncu --set full, profiles/traffic.json)",
        "peak_basis": f"{SM_COUNT} SMs x {sm_max:.0f} MHz (sm_max) x {LDS_LANES_PER_CLK} lane-lookups/clk/SM / "
                      f"(16*Nr lookups per 16 B)",
        "frac_at_measured_clock": (achieved / compute_peak_gbs(key_bytes, clocks["sm_mhz"])) if clocks.get("sm_mhz") else None,
        "hbm_payload_peak": peaks["hbm_gbs"] / (2 + 16.0 / PB),
        "hbm_peak_source": ("fallback 6650 GB/s (no MEASURED_PEAKS.json)" if peaks.get("_fallback")
                            else "MEASURED_PEAKS.json"),
        "hbm_frac": achieved / (peaks["hbm_gbs"] / (2 + 16.0 / PB)),
        "kernel": kernel, "algorithmic_bytes_per_launch": bytes_launch, "launches_per_step": launches_per_step,
        "avg_launch_ms": 1e3 * avg_launch_max,
        "page_loads": "LDG" if os.environ.get("KG_TEXIN") == "0" else "texture pipe (TLD)",
    }
    return {
        "workload": desc, "name": workload, "value": value, "unit": "GB/s", "ms_per_step": 1e3 * elapsed_max / steps,
        "steps": steps, "warmup": warmup, "scaling": scaling, "n_pages_per_gpu": n, "n_pages_total":
            n_total * (ctx.world if scaling == "weak" else 1), "key_bits": 8 * key_bytes,
        "dir": "decrypt" if direction else "encrypt", "mode": "ecb" if mode else "cbc", "in_place": in_place,
        "roofline": roof, "e2e": e2e, "check": check, "clocks": clocks, "gpu_launches": launches_all,
        "wall_s_timed": t_wall,
        "l2": (f"no flush: each step reads {n * PB / 2**20:.0f} MiB" +
               ("" if in_place else f" and writes {n * PB / 2**20:.0f} MiB") + " per GPU, > 126 MB L2"),
    }


def c4_sweep(ctx, args):
    """configs[3] on rank 0 (one GPU): caller-observed latency of ONE request
    (submit -> kg_wait returns) from 1 page to 1 GiB, HBM and pinned host
    (the library's default host path), beside the oracle and single-core
    OpenSSL at the same size; crossover = smallest size from which the GPU's
    p50 stays at or below the CPU's (a tie counts for the GPU)."""
    import oracle
    import paper_1305_3345_b200 as kg
    torch = ctx.torch
    kmax = args.sweep_kmax
    nmax = 1 << kmax
    key = synth.make_key(16)
    kg.set_key(0, key)
    threads = len(os.sched_getaffinity(0))
    data = synth.make_pages(nmax, PB)
    ivs_np = synth.make_ivs(nmax)
    dx = torch.from_numpy(data).cuda()
    div = torch.from_numpy(ivs_np).cuda()
    dout = torch.empty_like(dx)
    hx = kg.alloc_pinned(nmax * PB)
    hx.copy_(torch.from_numpy(data))
    hout = kg.alloc_pinned(nmax * PB)
    hiv = kg.alloc_pinned(16 * nmax)
    hiv.copy_(torch.from_numpy(ivs_np))
    s = torch.cuda.current_stream()
    try:
        from cryptography.hazmat.primitives.ciphers import Cipher, algorithms, modes
    except Exception:  # noqa: BLE001
        Cipher = None

    def lat(fn, reps, pct=False):
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            fn()
            ts.append(time.perf_counter() - t0)
        if not pct:
            return 1e6 * statistics.median(ts)
        q = np.percentile(np.array(ts) * 1e6, [10, 50, 90])
        return [round(float(x), 2) for x in q]

    rows = []
    for k in range(kmax + 1):
        n = 1 << k
        reps = 50 if n * PB < (1 << 20) else 10    # >= 50 below 1 MiB, >= 10 above
        row = {"pages": n}
        for name, (a, b, c) in (("hbm", (dx, dout, div)), ("pinned", (hx, hout, hiv))):
            def f():
                kg.wait(kg.submit_pages(1, 0, a, b, n, PB, c, 0, s))
            for _ in range(3):
                f()
            p10, p50, p90 = lat(f, reps, pct=True)
            row[f"{name}_us"] = p50
            row[f"{name}_us_p10_p90"] = [p10, p90]
            row[f"{name}_gbs"] = round(n * PB / (p50 * 1e-6) / 1e9, 3)
        if n <= args.sweep_nsk_pages:
            kg.nsk_start(16, kg.NSK_DIRECT | kg.NSK_NOCAL, 5000)

            def g():
                kg.wait(kg.submit_pages(1, 0, dx, dout, n, PB, div, 0, s))
            for _ in range(3):
                g()
            row["nsk_hbm_us"] = round(lat(g, reps), 2)
            kg.nsk_stop()
        c_np = data[: n * PB]
        iv_np = ivs_np[: 16 * n]
        if n <= 64:
            row["oracle_1t_us"] = round(lat(lambda: oracle.pages(1, 0, key, c_np, n, PB, iv_np, threads=1),
                                            5 if n < 16 else 2), 1)
        if n <= 1024:
            row["oracle_T_us"] = round(lat(lambda: oracle.pages(1, 0, key, c_np, n, PB, iv_np, threads=threads),
                                           5 if n < 64 else 2), 1)
        if Cipher is not None and n <= 4096:
            cb, ivb = c_np.tobytes(), iv_np.tobytes()

            def ossl():
                for p in range(n):
                    Cipher(algorithms.AES(key), modes.CBC(ivb[16 * p:16 * p + 16])).decryptor().update(
                        cb[p * PB:(p + 1) * PB])
            row["openssl_1core_us"] = round(lat(ossl, 5 if n < 256 else 2), 1)
        rows.append(row)
    # Row f2: the size-based dispatcher as a caller sees it.  kg_nsk_start
    # calibrates the NSK/launch crossover on the device (PAPER.md:493-495's
    # "calibrate it using microbenchmarks at boot time"); requests up to the
    # chosen size go to the resident kernel, larger ones are launched on the SMs
    # it leaves free.
    kg.nsk_start(16, kg.NSK_DIRECT, 5000)
    try:
        cal = kg.nsk_calibration()
        dispatch = {"threshold_bytes": kg.dispatch_threshold(cal),
                    "calibration": [{"bytes": b, "nsk_us": round(nu, 2), "launch_us": round(lu, 2)} for b, nu, lu in cal],
                    "rule": "largest calibrated size below the first at which the launch is faster (tie -> NSK)"}
        for row in rows:
            n = row["pages"]

            def g2():
                kg.wait(kg.submit_pages(1, 0, dx, dout, n, PB, div, 0, s))
            for _ in range(3):
                g2()
            row["auto_hbm_us"] = round(lat(g2, 50 if n * PB < (1 << 20) else 10), 2)
    finally:
        kg.nsk_stop()
    kg.free_pinned(hx)
    kg.free_pinned(hout)
    kg.free_pinned(hiv)
    del dx, dout, div
    torch.cuda.empty_cache()

    def crossover(gk, ck):
        pts = [r for r in rows if gk in r and ck in r]
        for r in pts:
            if all(q[gk] <= q[ck] for q in pts if q["pages"] >= r["pages"]):
                return {"bytes": r["pages"] * PB, "measured_pages": [pts[0]["pages"], pts[-1]["pages"]]}
        return {"bytes": None, "measured_pages": [pts[0]["pages"], pts[-1]["pages"]] if pts else None}

    cross = {}
    for gk in ("hbm_us", "pinned_us", "nsk_hbm_us", "auto_hbm_us"):
        for ck in ("oracle_1t_us", "oracle_T_us", "openssl_1core_us"):
            cross[f"{gk[:-3]} vs {ck[:-3]}"] = crossover(gk, ck)
    return {"workload": "C4 request batch-size sweep: AES-128-CBC decrypt, one request of 2^k 4 KiB pages, "
                        f"k = 0..{kmax}; p50 latency in us (submit -> kg_wait returns, through Python), "
                        "p10/p90 and GB/s at the p50 for the launch paths",
            "oracle_threads": threads, "rows": rows, "crossover": cross, "nsk_dispatch": dispatch,
            "note": "crossover = smallest size from which the GPU p50 stays <= the CPU's (tie -> GPU); "
                    "openssl = single-core AES-NI via `cryptography`, context not the oracle; "
                    "auto = the NSK running with its start-up calibrated dispatch (row f2); "
                    "the paper: GPU faster from 8 KB (PAPER.md:460-463)"}


def c1_latency(ctx, args):
    """configs[0] (C1): AES-128-CBC encrypt, then decrypt, of 16 seeded 4 KiB
    pages in HBM; caller-observed latency of each direction (p10/p50/p90 over
    200 requests) and the round trip; plus SP 800-38A F.2.1/F.2.2 (CBC-AES128
    encrypt/decrypt) as one 64-byte page each, against the standard's values."""
    import paper_1305_3345_b200 as kg
    torch = ctx.torch
    n = 16
    kg.set_key(5, synth.make_key(16))
    x = torch.from_numpy(synth.make_pages(n, PB)).cuda()
    iv = torch.from_numpy(synth.make_ivs(n)).cuda()
    c = torch.empty_like(x)
    back = torch.empty_like(x)
    s = torch.cuda.current_stream()
    out = {"workload": "C1: AES-128-CBC encrypt then decrypt of 16 x 4 KiB pages (64 KiB), HBM, per-page IVs"}
    for name, (d, a, b) in (("encrypt", (0, x, c)), ("decrypt", (1, c, back))):
        ts = []
        for r in range(210):
            t0 = time.perf_counter()
            kg.wait(kg.submit_pages(d, 0, a, b, n, PB, iv, 5, s))
            if r >= 10:
                ts.append(1e6 * (time.perf_counter() - t0))
        out[f"{name}_us_p10_p50_p90"] = [round(float(v), 2) for v in np.percentile(ts, [10, 50, 90])]
    torch.cuda.synchronize()
    out["round_trip_equal"] = bool(torch.equal(back, x))
    key = bytes.fromhex("2b7e151628aed2a6abf7158809cf4f3c")
    pt = bytes.fromhex("6bc1bee22e409f96e93d7e117393172aae2d8a571e03ac9c9eb76fac45af8e51"
                       "30c81c46a35ce411e5fbc1191a0a52eff69f2445df4f9b17ad2b417be66c3710")
    ct = bytes.fromhex("7649abac8119b246cee98e9b12e9197d5086cb9b507219ee95db113a917678b2"
                       "73bed6b8e3c1743b7116e69e222295163ff1caa1681fac09120eca307586e1a7")
    kg.set_key(6, key)
    tiv = torch.arange(16, dtype=torch.uint8).cuda()
    tp = torch.frombuffer(bytearray(pt), dtype=torch.uint8).cuda()
    tc = torch.empty_like(tp)
    kg.wait(kg.submit_pages(0, 0, tp, tc, 1, 64, tiv, 6, s))
    tb = torch.empty_like(tp)
    kg.wait(kg.submit_pages(1, 0, tc, tb, 1, 64, tiv, 6, s))
    torch.cuda.synchronize()
    out["sp800_38a_f21_encrypt_ok"] = tc.cpu().numpy().tobytes() == ct
    out["sp800_38a_f22_decrypt_ok"] = tb.cpu().numpy().tobytes() == pt
    return out


def run_ours(args):
    import torch

    import paper_1305_3345_b200 as kg

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world != args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} but WORLD_SIZE={world}: refusing to report a mislabelled "
                                   "n_gpus", "rank": rank, "world": world}), flush=True)
        return 2
    if not torch.cuda.is_available():
        print(json.dumps({"error": "no CUDA device", "rank": rank, "world": world}), flush=True)
        return 1
    ctx = Ctx(args)
    kg.init(ctx.dev)

    head = run_config(ctx, args, args.workload, args.steps, args.warmup)
    extras = {}
    if args.workload == "c2" and args.extra != "none":
        names = DEFAULT_EXTRA if args.extra == "default" else tuple(x for x in args.extra.split(",") if x)
        for name in names:
            if name not in WORKLOADS or name == args.workload:
                continue
            extras[name] = run_config(ctx, args, name, args.steps, args.warmup)
    sweep = c1 = None
    if ctx.world == 1 and not args.no_sweep and args.workload == "c2":
        c1 = c1_latency(ctx, args)
        sweep = c4_sweep(ctx, args)

    if ctx.rank != 0:
        if ctx.dist:
            ctx.dist.barrier()
            ctx.dist.destroy_process_group()
        return 0

    line = {
        "metric": METRIC, "value": head["value"], "unit": "GB/s", "n_gpus": ctx.world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": head["ms_per_step"], "higher_is_better": True,
        "scaling": head["scaling"], "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": head["workload"], "name": args.workload, "n_pages_per_gpu": head["n_pages_per_gpu"],
                   "page_bytes": PB, "key_bits": head["key_bits"], "dir": head["dir"], "mode": head["mode"],
                   "residency": "hbm", "in_place": head["in_place"], "l2": head["l2"],
                   "parallelism": f"page-range x{ctx.world}" if ctx.world > 1 else "1 GPU",
                   "timing": (f"{args.warmup} warm-up steps, barrier + synchronize, {args.queue_ahead_steps} untimed "
                              f"queue-ahead steps, then CUDA events around exactly {args.steps} back-to-back steps "
                              "on the launching stream; synchronize; max over ranks")},
        "roofline": head["roofline"],
        "e2e": head["e2e"],
        "gpu_launches": head["gpu_launches"],
        "check": head["check"],
        "clocks": head["clocks"],
        "clocks_all_timed_regions": merge_clocks([head["clocks"]] + [c["clocks"] for c in extras.values()]),
        "comm": ctx.comm,
        "wall_s_timed": head["wall_s_timed"],
        "configs": extras,
    }
    if c1:
        line["c1"] = c1
    if sweep:
        line["c4_sweep"] = sweep
    if ctx.world == 1 and not args.no_cpu_baseline:
        threads = len(os.sched_getaffinity(0))
        n_total, key_bytes, direction = WORKLOADS[args.workload][:3]
        gbs, npg, dt = oracle_rate(n_total, key_bytes, direction, args.cpu_seconds, threads)
        g1, n1, d1 = oracle_rate(n_total, key_bytes, direction, args.cpu_seconds / 2, 1)
        line["cpu_baseline"] = {
            "value": gbs, "unit": "GB/s", "cores": threads, "kind": "oracle",
            "sample": f"{npg} seeded 4 KiB pages ({npg * PB / 2**20:.1f} MiB) of the same workload, "
                      f"{threads} pthreads, {dt:.1f} s",
            "one_thread": {"value": g1, "unit": "GB/s", "cores": 1,
                           "sample": f"{n1} seeded 4 KiB pages ({n1 * PB / 2**20:.1f} MiB), 1 thread, {d1:.1f} s"}}
        line["context"] = {"openssl_aesni_1core": openssl_rate(key_bytes, direction)}
    print(json.dumps(line), flush=True)
    if args.csv:
        write_csv(args.csv, line)
    if ctx.dist:
        ctx.dist.barrier()
        ctx.dist.destroy_process_group()
    return 0


CSV_COLUMNS = ("config", "dir", "key_bits", "residency", "gpus", "n_pages", "page_bytes", "latency_us_p50", "gbps",
               "roofline_gbps", "pct_roofline", "sm_mhz_median", "host_cores")


def csv_rows(line):
    """The line's measurements as rows with SURVEY.md §5's columns (SPEC.md:470's
    experiment CSV, extended): one row per config and residency (hbm = the
    device-timed value; pinned = its e2e), one per C4 sweep point and path.
    latency_us_p50 is the per-step time for the configs (K back-to-back steps)
    and the caller-observed p50 for the sweep; roofline_gbps is the lookup bound
    (pinned rows: the duplex host link measured in the same run)."""
    rows = []
    mhz = (line.get("clocks") or {}).get("sm_mhz")
    cores = (line.get("cpu_baseline") or {}).get("cores", "")
    heads = [(line["config"]["name"], line)] + sorted((line.get("configs") or {}).items())
    for name, c in heads:
        cfg = c.get("config", c)
        dirn, kbits = cfg.get("dir", c.get("dir")), cfg.get("key_bits", c.get("key_bits"))
        n = cfg.get("n_pages_per_gpu", c.get("n_pages_per_gpu"))
        roof = c["roofline"]
        rows.append({"config": name, "dir": dirn, "key_bits": kbits, "residency": "hbm", "gpus": line["n_gpus"],
                     "n_pages": n, "page_bytes": PB, "latency_us_p50": round(1e3 * c["ms_per_step"], 3),
                     "gbps": round(c["value"], 3), "roofline_gbps": round(roof["peak"], 3),
                     "pct_roofline": round(100 * roof["frac"], 2),
                     "sm_mhz_median": (c.get("clocks") or {}).get("sm_mhz", mhz), "host_cores": cores})
        e = c.get("e2e")
        if e:
            link = e.get("link_duplex_aggregate_gbs_per_direction")
            rows.append({"config": name, "dir": dirn, "key_bits": kbits, "residency": "pinned", "gpus": line["n_gpus"],
                         "n_pages": n, "page_bytes": PB,
                         "latency_us_p50": round(1e3 * e["step_ms_min_median_max"][1], 3)
                         if e.get("step_ms_min_median_max") else "",
                         "gbps": round(e["value"], 3), "roofline_gbps": round(link, 3) if link else "",
                         "pct_roofline": round(100 * e["value"] / link, 2) if link else "",
                         "sm_mhz_median": (c.get("clocks") or {}).get("sm_mhz", mhz), "host_cores": cores})
    sw = line.get("c4_sweep")
    if sw:
        peak = compute_peak_gbs(16, float((line.get("clocks") or {}).get("sm_max_mhz") or 1965.0))
        link = (line.get("e2e") or {}).get("link_duplex_aggregate_gbs_per_direction")
        threads = {"oracle_1thread": 1, "oracle_threads": sw.get("oracle_threads", cores), "openssl_1core": 1}
        paths = (("hbm_us", "hbm"), ("pinned_us", "pinned"), ("nsk_hbm_us", "hbm_nsk"), ("auto_hbm_us", "hbm_auto"),
                 ("oracle_1t_us", "oracle_1thread"), ("oracle_T_us", "oracle_threads"),
                 ("openssl_1core_us", "openssl_1core"))
        for r in sw["rows"]:
            for key, res in paths:
                if key not in r:
                    continue
                gbs = r["pages"] * PB / (r[key] * 1e-6) / 1e9
                gpu = res.startswith(("hbm", "pinned"))
                bound = (link if res == "pinned" else peak) if gpu else None
                rows.append({"config": "c4", "dir": "decrypt", "key_bits": 128, "residency": res, "gpus": 1,
                             "n_pages": r["pages"], "page_bytes": PB, "latency_us_p50": r[key], "gbps": round(gbs, 3),
                             "roofline_gbps": round(bound, 3) if bound else "",
                             "pct_roofline": round(100 * gbs / bound, 2) if bound else "",
                             "sm_mhz_median": mhz if gpu else "", "host_cores": "" if gpu else threads[res]})
    return rows


def write_csv(path, line):
    import csv
    with open(path, "w", newline="") as f:
        w = csv.DictWriter(f, fieldnames=CSV_COLUMNS)
        w.writeheader()
        for r in csv_rows(line):
            w.writerow(r)


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def self_launch(args, argv):
    """--gpus N > 1 without a launcher: re-run this script under
    torch.distributed.run, one rank per GPU (NCCL), rendezvous on 127.0.0.1.
    NCCL_DEBUG=INFO (INIT subsystem) unless the caller set it, so the log
    shows the communicator's rank count."""
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + argv
    return subprocess.call(cmd, env=env)


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--extra", default="default",
                    help="comma list of extra workloads in the same line (with --workload c2); 'none' to skip")
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--e2e-depth", type=int, default=3,
                    help="e2e: batches the caller keeps in flight (out-of-place workloads; 1 = submit, wait, repeat)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-check", action="store_true")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--sweep-kmax", type=int, default=18)
    ap.add_argument("--sweep-nsk-pages", type=int, default=256)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--queue-ahead-steps", type=int, default=3,
                    help="untimed steps enqueued after the barrier, right before the start event (0: none)")
    ap.add_argument("--csv", default="",
                    help="also write the line's measurements as CSV rows (SURVEY.md §5 columns) to this path")
    ap.add_argument("--ref-step-seconds", type=float, default=0.0,
                    help="reference arm: oracle seconds per step (default: sized so the run takes ~2.5 min)")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_launch(args, argv)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
