#!/usr/bin/env python
"""bench.py -- AES-CBC page-crypto throughput on B200 (BASELINE.json metric).

Default workload (N=1, the configuration BASELINE.json's metric is quoted on,
configs[1]): "eCryptfs-shaped read": AES-128-CBC DECRYPT of a 256 MiB batch
of 65,536 independent 4 KiB pages with per-page IVs, HBM-resident.  One
step = one pass of the whole hot path over one batch: kg_submit_pages
(validate, snapshot key, enqueue) -> the decrypt kernel -> completion ticket
(kg_wait).  Keys are expanded once (kg_set_key), outside the timed region
("key expansion once per key", BASELINE.json:5).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c2|c3|c5]
  torchrun ... bench.py --gpus N     (one rank per GPU, NCCL; weak scaling:
                                      every rank decrypts its own 256 MiB)
  python bench.py --impl reference   (the oracle on the host cores: a
                                      bounded sample of the same workload)

Prints ONE JSON line on rank 0.  `value` = payload GB/s (10^9 page bytes per
second, IVs excluded) over all ranks, device-timed with CUDA events on the
launching stream, max over ranks.  `e2e` = the same metric through the C ABI
with pinned HOST buffers (H2D + kernel + D2H inside the timed region, i.e.
the pinned-host-resident figure of the metric).  See DESIGN.md §Measurement.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
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
WORKLOADS = {
    # name: (n_pages per rank, key_bytes, dir, in_place, description)
    "c2": (65536, 16, 1, False, "C2 eCryptfs-shaped read: AES-128-CBC decrypt, 65,536 x 4 KiB pages (256 MiB) per GPU, HBM-resident, out-of-place"),
    "c3": (262144, 32, 0, False, "C3 eCryptfs-shaped write: AES-256-CBC encrypt (page-parallel chains), 262,144 x 4 KiB pages (1 GiB) per GPU, HBM-resident"),
    "c5": (16777216, 16, 1, True, "C5: AES-128-CBC decrypt of 64 GiB (16,777,216 x 4 KiB pages) page-range sharded over the ranks, HBM-resident, in place"),
    # not BASELINE configs: the paper's own ECB mode (row f1) and mixed-key batches
    "ecb_dec": (65536, 16, 1, False, "AES-128-ECB decrypt (the paper's mode, PAPER.md:448-450), 65,536 x 4 KiB pages, HBM"),
    "ecb_enc": (65536, 16, 0, False, "AES-128-ECB encrypt (the paper's mode, PAPER.md:448-450), 65,536 x 4 KiB pages, HBM"),
    "c2_keyed": (65536, 16, 1, False, "C2 with a key id per page (8 AES-128 keys, uniform), HBM, out-of-place"),
    "c3_keyed": (262144, 32, 0, False, "C3 with a key id per page (8 AES-256 keys, uniform), HBM, out-of-place"),
    "c2_inplace": (65536, 16, 1, True, "C2 in place (AES-128-CBC decrypt, 65,536 x 4 KiB pages), HBM"),
    "ecb_dec_inplace": (65536, 16, 1, True, "AES-128-ECB decrypt in place, 65,536 x 4 KiB pages, HBM"),
}
KEYED = ("c2_keyed", "c3_keyed")
MODE_OF = {"ecb_dec": 1, "ecb_enc": 1, "ecb_dec_inplace": 1}
SM_COUNT = 148
LDS_LANES_PER_CLK = 32      # lane-lookups/clk/SM (B300_MICROARCH.md "smem crossbar 128/N B/cyc/SM"; tools/pipes.cu measures it)


def nr_of(key_bytes):
    return {16: 10, 24: 12, 32: 14}[key_bytes]


def compute_peak_gbs(key_bytes, sm_mhz, sms=SM_COUNT):
    """T-table compute ceiling in payload GB/s: 16*Nr lane-lookups per 16-byte
    block at LDS_LANES_PER_CLK per SM per clock."""
    return sms * sm_mhz * 1e6 * LDS_LANES_PER_CLK * 16.0 / (16.0 * nr_of(key_bytes)) / 1e9


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
    """pynvml sampling of SM clock + throttle reasons during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, index, period=0.005):
        self.ok = False
        self.samples, self.reasons = [], set()
        self.period = period
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:  # noqa: BLE001
            self.max_mhz = None
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def duplex_link_gbs(torch, h_a, h_b, nbytes=128 << 20, reps=5):
    """Measured concurrent H2D + D2H pinned copy bandwidth per direction (the
    pinned-host path's roofline: every payload byte crosses the link both ways)."""
    nbytes = min(nbytes, h_a.numel(), h_b.numel())
    d_a = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    d_b = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    best = None
    for _ in range(reps):
        torch.cuda.synchronize()
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
        best = t if best is None else min(best, t)
    return nbytes / best / 1e9


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


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


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    n_pages, key_bytes, direction, _, desc = WORKLOADS[args.workload]
    threads = len(os.sched_getaffinity(0))
    per_step = args.ref_step_seconds or max(0.5, min(10.0, 150.0 / max(1, args.steps + args.warmup)))
    import oracle
    key = synth.make_key(key_bytes)
    # calibrate the per-step sample
    _, n, dt = oracle_rate(n_pages, key_bytes, direction, per_step, threads)
    data = synth.make_pages(n, PB)
    ivs = synth.make_ivs(n)
    for _ in range(args.warmup):
        oracle.pages(direction, 0, key, data, n, PB, ivs, threads=threads)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.pages(direction, 0, key, data, n, PB, ivs, threads=threads)
        times.append(time.perf_counter() - t0)
    total = sum(times)
    gbs = n * PB * args.steps / total / 1e9
    sample = f"{n} of the workload's {n_pages} 4 KiB pages per step ({n * PB / 2**20:.1f} MiB), {threads} pthreads"
    line = {
        "impl": "reference", "metric": METRIC, "value": gbs, "unit": "GB/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": desc, "n_pages": n_pages, "page_bytes": PB, "key_bits": 8 * key_bytes,
                   "dir": "decrypt" if direction else "encrypt", "sampled_pages_per_step": n},
        "cpu_baseline": {"value": gbs, "unit": "GB/s", "cores": threads, "kind": "oracle", "sample": sample},
        "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- our arm
def run_ours(args):
    import torch

    import paper_1305_3345_b200 as kg

    world, rank, local = dist_env()
    if not torch.cuda.is_available():
        print(json.dumps({"error": "no CUDA device"}))
        return 1
    # one process per GPU; KG_BENCH_SHARE_GPU=1 (testing the N>1 code path on a
    # one-GPU box) maps ranks onto the available devices and uses gloo
    share = os.environ.get("KG_BENCH_SHARE_GPU") == "1"
    dev = local % torch.cuda.device_count() if share else local
    torch.cuda.set_device(dev)
    dist = None
    red_dev = "cuda"
    if world > 1:
        import torch.distributed as dist
        if share:
            dist.init_process_group("gloo")
            red_dev = "cpu"
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
    kg.init(dev)
    n_total, key_bytes, direction, in_place, desc = WORKLOADS[args.workload]
    if args.workload == "c5":
        lo, hi = synth.shard(n_total, rank, world)   # strong scaling: 64 GiB split by page range
        scaling = "strong"
    else:
        lo, hi = 0, n_total                           # weak scaling: every rank its own batch
        scaling = "weak"
    n = hi - lo
    key = synth.make_key(key_bytes)
    kg.set_key(0, key)
    mode = MODE_OF.get(args.workload, kg.MODE_CBC)
    keyed = args.workload in KEYED
    if keyed:
        for i in range(8):
            kg.set_key(i, synth.make_key(key_bytes, seed=synth.KEY_SEED + 100 + i))
    stream = torch.cuda.current_stream()

    # inputs: seeded pages (C2/C3: the full batch; C5: periodic M-page pattern)
    M = 65537
    if args.workload == "c5":
        pat = torch.from_numpy(synth.make_pages(M, PB)).cuda().view(M, PB)
        ivp = torch.from_numpy(synth.make_ivs(M)).cuda().view(M, 16)
        x = torch.empty((n, PB), dtype=torch.uint8, device="cuda")
        ivs = torch.empty((n, 16), dtype=torch.uint8, device="cuda")
        for s in range(0, n, M):
            e = min(n, s + M)
            idx = (torch.arange(s, e, device="cuda") + lo) % M
            x[s:e] = pat[idx]
            ivs[s:e] = ivp[idx]
        del pat, ivp
        x = x.view(-1)
        ivs = ivs.view(-1)
    else:
        x = torch.from_numpy(synth.make_pages(n, PB, first_page=lo)).cuda()
        ivs = torch.from_numpy(synth.make_ivs(n, first_page=lo)).cuda()
    out = x if in_place else torch.empty_like(x)
    key_ids = None
    if keyed:
        key_ids = torch.from_numpy((synth.stream_bytes(synth.KEY_SEED + 7, 2 * n).view(np.uint16) % 8)
                                   .astype(np.int16)).cuda()
    torch.cuda.synchronize()

    def step():
        if keyed:
            return kg.submit_pages_keyed(direction, mode, x, out, n, PB, ivs, key_ids, key_bytes, stream)
        return kg.submit_pages(direction, mode, x, out, n, PB, ivs if mode == kg.MODE_CBC else None, 0, stream)

    # warm-up (also loads the module lazily)
    for _ in range(args.warmup):
        kg.wait(step())
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    l0 = kg.launch_count()
    with ClockSampler(dev) as clk:
        t_wall0 = time.perf_counter()
        tickets = []
        for i in range(args.steps):
            if args.step_events or i == 0:
                starts[i].record(stream)
            tickets.append(step())
            if args.step_events or i == args.steps - 1:
                ends[i].record(stream)
        for t in tickets:
            kg.wait(t)
        torch.cuda.synchronize()
        t_wall = time.perf_counter() - t_wall0
    launches = kg.launch_count() - l0
    elapsed = starts[0].elapsed_time(ends[-1]) / 1e3                   # s, device-timed
    if args.step_events:
        per_launch = [s.elapsed_time(e) / 1e3 for s, e in zip(starts, ends)]
        avg_launch = sum(per_launch) / max(launches, len(per_launch))
    else:
        # launches back to back on one stream; a step is one launch, or several
        # page windows when the input exceeds one texture (C5)
        avg_launch = elapsed / max(launches, args.steps)
    if dist:
        t = torch.tensor([elapsed, avg_launch], dtype=torch.float64, device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed, avg_launch = float(t[0]), float(t[1])
    bytes_step = n * PB
    total_bytes = bytes_step * args.steps * (world if scaling == "weak" else 1)
    if scaling == "strong":
        total_bytes = n_total * PB * args.steps
    value = total_bytes / elapsed / 1e9
    clocks = clk.summary()

    # correctness check outside the timed region (every rank, SUM over ranks):
    # one more step, then S sampled output pages go back through the inverse
    # operation on the GPU and must reproduce the step's input pages.
    check = None
    if not args.no_check:
        S = min(n, 1024)
        gen = torch.Generator().manual_seed(1305 + rank)
        idx = torch.randperm(n, generator=gen)[:S].sort().values.cuda()
        xv = x.view(n, PB)
        before = xv[idx].clone()
        kg.wait(step())
        torch.cuda.synchronize()
        after = out.view(n, PB)[idx].contiguous()
        iv_s = ivs.view(n, 16)[idx].contiguous().view(-1) if mode == kg.MODE_CBC else None
        back = torch.empty_like(after)
        inv = 1 - direction
        if keyed:
            kid_s = key_ids[idx].contiguous()
            kg.wait(kg.submit_pages_keyed(inv, mode, after.view(-1), back.view(-1), S, PB, iv_s, kid_s, key_bytes, stream))
        else:
            kg.wait(kg.submit_pages(inv, mode, after.view(-1), back.view(-1), S, PB, iv_s, 0, stream))
        torch.cuda.synchronize()
        bad = torch.tensor([float((back != before).any(dim=1).sum()), float(S)], dtype=torch.float64, device=red_dev
                           if dist else "cpu")
        if dist:
            dist.all_reduce(bad, op=dist.ReduceOp.SUM)
        check = {"sampled_pages": int(bad[1]), "mismatched_pages": int(bad[0]),
                 "method": "one extra step; sampled output pages through the inverse operation on the GPU "
                           "must give back the step's input pages (parity vs the oracle: tests/)"}

    # secondary: e2e through the C ABI with pinned HOST buffers (H2D + compute + D2H timed)
    e2e = None
    if args.workload in ("c2", "c3", "c5") and not args.no_e2e:
        big = args.workload == "c5"            # 64 GiB: NUMA-local pinned shard, in place
        e_steps = max(1, min(args.steps, 2 if big else args.e2e_steps))
        if big:
            hx = kg.alloc_pinned(n * PB)
            hx.copy_(x)
            hiv = kg.alloc_pinned(16 * n)
            hiv.copy_(ivs)
            hout = hx
            residency = "pinned host shard (kg_alloc_pinned: cudaHostAlloc from GPU-local CPUs), in place"
        else:
            hx = torch.empty(n * PB, dtype=torch.uint8).pin_memory()
            hx.copy_(x.cpu())
            hiv = ivs.cpu().pin_memory()
            hout = hx if in_place else torch.empty_like(hx).pin_memory()
            residency = "pinned host (cudaHostAlloc via torch pin_memory)"
        for _ in range(1 if big else 2):
            kg.wait(kg.submit_pages(direction, kg.MODE_CBC, hx, hout, n, PB, hiv, 0, stream))
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        step_ms = []
        t0 = time.perf_counter()
        for _ in range(e_steps):
            ts = time.perf_counter()
            kg.wait(kg.submit_pages(direction, kg.MODE_CBC, hx, hout, n, PB, hiv, 0, stream))
            step_ms.append((time.perf_counter() - ts) * 1e3)
        te = time.perf_counter() - t0
        if dist:
            tt = torch.tensor([te], dtype=torch.float64, device=red_dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            te = float(tt[0])
        total_e2e = (n_total * PB if scaling == "strong" else bytes_step * world) * e_steps
        e2e = {"value": total_e2e / te / 1e9, "unit": "GB/s",
               "h2d_bytes_per_step": bytes_step + 16 * n, "d2h_bytes_per_step": bytes_step,
               "steps": e_steps, "residency": residency,
               "step_ms_min_median_max": [round(min(step_ms), 3), round(sorted(step_ms)[len(step_ms) // 2], 3),
                                          round(max(step_ms), 3)]}
        # host-link roofline for this path: pinned H2D and D2H copy engines at once
        link = duplex_link_gbs(torch, hx, hout)
        e2e["link_duplex_gbs_per_direction"] = link
        e2e["link_frac"] = (e2e["value"] / world) / link if link else None
        if big:
            kg.free_pinned(hx)
            kg.free_pinned(hiv)
        del hx, hout, hiv

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return 0

    peaks = load_peaks()
    sm_max = float(clocks.get("sm_max_mhz") or peaks.get("sm_max_mhz", 1965.0))
    launches_per_step = max(1, launches // args.steps)
    bytes_launch = bytes_step / launches_per_step
    achieved = bytes_launch / avg_launch / 1e9
    peak = compute_peak_gbs(key_bytes, sm_max)
    roof = {
        "bound": "alu", "pipe": "lds (shared-memory T-table lookups: 16*Nr lane-lookups per 16-byte block)",
        "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
        "traffic": load_traffic(args.workload),
        "traffic_unit": "DRAM bytes per launch (ncu --set full, profiles/traffic.json)",
        "peak_basis": f"{SM_COUNT} SMs x {sm_max:.0f} MHz (sm_max) x {LDS_LANES_PER_CLK} lane-lookups/clk/SM / (16*Nr lookups per 16 B)",
        "frac_at_measured_clock": (achieved / compute_peak_gbs(key_bytes, clocks["sm_mhz"])) if clocks.get("sm_mhz") else None,
        "hbm_payload_peak": peaks["hbm_gbs"] / (2 + 16.0 / PB),
        "hbm_peak_source": ("fallback 6650 GB/s (no MEASURED_PEAKS.json)" if peaks.get("_fallback")
                            else "MEASURED_PEAKS.json"),
        "hbm_frac": achieved / (peaks["hbm_gbs"] / (2 + 16.0 / PB)),
        "kernel": (("kg_keyed_chain" if (direction == 0 and mode == kg.MODE_CBC) else "kg_keyed_pair") if keyed
                   else "kg_blockpar" if (direction == 1 or mode == kg.MODE_ECB) else "kg_cbc_enc") + f"<Nr={nr_of(key_bytes)},{'dec' if direction else 'enc'},{'ecb' if mode else 'cbc'}>",
        "algorithmic_bytes_per_launch": bytes_launch,
        "launches_per_step": launches_per_step,
        "page_loads": "LDG" if os.environ.get("KG_TEXIN") == "0" else "texture pipe (TLD)",
    }
    line = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * elapsed / args.steps, "higher_is_better": True,
        "scaling": scaling, "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": desc, "n_pages_per_gpu": n, "page_bytes": PB, "key_bits": 8 * key_bytes,
                   "dir": "decrypt" if direction else "encrypt", "mode": "ecb" if mode else "cbc", "residency": "hbm",
                   "l2": f"no flush: each step reads {bytes_step / 2**20:.0f} MiB and writes "
                         f"{bytes_step / 2**20:.0f} MiB, > 126 MB L2",
                   "parallelism": f"page-range x{world}" if world > 1 else "1 GPU"},
        "roofline": roof,
        "e2e": e2e,
        "gpu_launches": launches,
        "check": check,
        "clocks": clocks,
        "wall_s_timed": t_wall,
    }
    if world == 1 and not args.no_cpu_baseline:
        threads = len(os.sched_getaffinity(0))
        gbs, npg, dt = oracle_rate(n_total, key_bytes, direction, args.cpu_seconds, threads)
        line["cpu_baseline"] = {"value": gbs, "unit": "GB/s", "cores": threads, "kind": "oracle",
                                "sample": f"{npg} seeded 4 KiB pages ({npg * PB / 2**20:.1f} MiB) of the same workload, "
                                          f"{threads} pthreads, {dt:.1f} s"}
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--e2e-steps", type=int, default=30)
    ap.add_argument("--step-events", action="store_true",
                    help="record a CUDA event pair around every step (serialises programmatic dependent launch)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-check", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--ref-step-seconds", type=float, default=0.0,
                    help="reference arm: oracle seconds per step (default: sized so the run takes ~2.5 min)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
