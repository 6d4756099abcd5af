#!/usr/bin/env python
"""Summarise an ncu report (.ncu-rep) into a small JSON/markdown record for
profiles/.  Runs here (no GPU needed): `ncu -i REP --page raw --csv`.

usage: python tools/ncu_summary.py REP.ncu-rep [--out profiles/NAME] [--payload BYTES]
"""
import argparse
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "Kernel Name", "gpu__time_duration.sum", "launch__grid_size", "launch__block_size",
    "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
    "sm__cycles_elapsed.avg.per_second", "smsp__cycles_active.avg",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_lg.sum" , "l1tex__data_pipe_lsu_wavefronts.sum",
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum",
    "sm__inst_executed.sum", "sm__inst_executed.avg.per_cycle_active", "smsp__inst_executed.avg.per_cycle_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed_op_shared_ld.sum", "smsp__sass_inst_executed_op_shared_ld.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "achieved_occupancy",
    "smsp__average_warp_latency_issue_stalled_mio_throttle", "smsp__average_warp_latency_issue_stalled_short_scoreboard",
    "smsp__pcsamp_warps_issue_stalled_mio_throttle", "smsp__pcsamp_warps_issue_stalled_short_scoreboard",
    "smsp__pcsamp_warps_issue_stalled_lg_throttle", "smsp__pcsamp_warps_issue_stalled_long_scoreboard",
    "smsp__pcsamp_warps_issue_stalled_selected", "smsp__pcsamp_warps_issue_stalled_not_selected",
    "smsp__pcsamp_warps_issue_stalled_wait", "smsp__pcsamp_warps_issue_stalled_math_pipe_throttle",
    "smsp__pcsamp_warps_issue_stalled_barrier", "smsp__pcsamp_warps_issue_stalled_dispatch_stall",
    "smsp__pcsamp_sample_count",
    "SM_A.TriageCompute.l1tex__data_pipe_lsu_wavefronts.avg", "SM_A.TriageCompute.l1tex__data_pipe_lsu_wavefronts_mem_lgds.avg",
    "SM_A.TriageCompute.l1tex__data_pipe_lsu_wavefronts_mem_shared.avg", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_st.sum",
    "memory_l1_wavefronts_shared", "memory_l1_wavefronts_shared_ideal", "smsp__inst_executed.sum",
    "sm__issue_active.avg.pct_of_peak_sustained_elapsed", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_elapsed",
]


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    header, units = rows[0], rows[1]
    return header, units, rows[2:]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--out")
    ap.add_argument("--payload", type=float, default=None, help="algorithmic payload bytes per launch")
    ap.add_argument("--all", action="store_true", help="dump every metric")
    a = ap.parse_args()
    header, units, rows = raw_rows(a.rep)
    recs = []
    for r in rows:
        d = dict(zip(header, r))
        u = dict(zip(header, units))
        if a.all:
            rec = {k: (d[k], u.get(k, "")) for k in header}
        else:
            rec = {k: (d[k], u.get(k, "")) for k in KEYS if k in d}
            for k in header:
                if k.startswith("smsp__pcsamp_warps_issue_stalled") and k not in rec and d[k] not in ("", "0"):
                    rec[k] = (d[k], u.get(k, ""))
        if a.payload:
            try:
                t = float(d["gpu__time_duration.sum"].replace(",", ""))
                unit = u.get("gpu__time_duration.sum", "ns")
                scale = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "nsecond": 1e-9, "msecond": 1e-3, "ms": 1e-3}.get(unit, 1e-9)
                rec["payload_GBps_at_ncu_time"] = (f"{a.payload / (t * scale) / 1e9:.2f}", "GB/s")
            except (KeyError, ValueError):
                pass
        recs.append(rec)
    js = json.dumps(recs, indent=1)
    if a.out:
        with open(a.out + ".json", "w") as f:
            f.write(js)
        with open(a.out + ".md", "w") as f:
            for i, rec in enumerate(recs):
                f.write(f"### launch {i}: {rec.get('Kernel Name', ('?',))[0][:120]}\n\n| metric | value | unit |\n|---|---|---|\n")
                for k, (v, un) in rec.items():
                    if k == "Kernel Name":
                        continue
                    f.write(f"| {k} | {v} | {un} |\n")
                f.write("\n")
    else:
        print(js)


if __name__ == "__main__":
    sys.exit(main())
