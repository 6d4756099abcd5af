"""bench.py on the GPU: the N>1 path launched the way the driver's command
line does it (--gpus 2, no external launcher: bench.py re-launches itself as
two ranks; KG_BENCH_SHARE_GPU=1 puts both ranks on this box's one GPU with a
gloo group), and the N=1 line's contract.  Every check is over every page."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _run(args, extra_env=None, timeout=900):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["PYTHONPATH"] = ROOT
    env.update(extra_env or {})
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                       timeout=timeout, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-3000:]
    return lines[0]


def _check_config(c, n_gpus):
    assert c["value"] > 0 and c["check"]["mismatched_pages"] == 0
    per_gpu = c["n_pages_per_gpu"] if "n_pages_per_gpu" in c else c["config"]["n_pages_per_gpu"]
    if c["scaling"] == "weak":
        assert c["check"]["pages"] == per_gpu * n_gpus
    assert 0 < c["roofline"]["frac"] < 1.05
    assert c["gpu_launches"] >= c["steps"] * n_gpus


def test_bench_two_ranks_self_launched():
    d = _run(["--gpus", "2", "--steps", "3", "--warmup", "3", "--extra", "c3", "--e2e-steps", "2"],
             {"KG_BENCH_SHARE_GPU": "1"})
    assert d["n_gpus"] == 2 and d["comm"]["world"] == 2 and d["comm"]["allreduce_sum_of_ones"] == 2
    assert d["check"]["mismatched_pages"] == 0 and d["check"]["pages"] == 2 * 65536
    _check_config(d, 2)
    _check_config(d["configs"]["c3"], 2)
    assert d["e2e"]["value"] > 0 and d["e2e"]["link_duplex_aggregate_gbs_per_direction"] > 0
    assert "cpu_baseline" not in d                       # rank 0 at N=1 only


def test_bench_one_gpu_line_contract(tmp_path):
    csv_path = tmp_path / "bench.csv"
    d = _run(["--steps", "5", "--warmup", "3", "--extra", "c3,c4_1gib", "--sweep-kmax", "6",
              "--sweep-nsk-pages", "4", "--cpu-seconds", "2", "--csv", str(csv_path)])
    import csv
    with open(csv_path) as f:
        rows = list(csv.DictReader(f))
    assert {(r["config"], r["residency"]) for r in rows} >= {("c2", "hbm"), ("c2", "pinned"), ("c3", "hbm"),
                                                             ("c4_1gib", "pinned"), ("c4", "hbm"), ("c4", "pinned")}
    assert abs(float(rows[0]["gbps"]) - d["value"]) < 1e-2
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks", "cpu_baseline"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 5 and d["dtype"] == "u8"
    _check_config(d, 1)
    for name in ("c3", "c4_1gib"):
        _check_config(d["configs"][name], 1)
        assert d["configs"][name]["e2e"]["value"] > 0
    assert d["cpu_baseline"]["one_thread"]["cores"] == 1
    rows = d["c4_sweep"]["rows"]
    assert [r["pages"] for r in rows] == [1 << k for k in range(7)]
    assert all(r["hbm_us"] > 0 and r["pinned_us"] > 0 for r in rows)
    assert all(r["hbm_us_p10_p90"][0] <= r["hbm_us"] <= r["hbm_us_p10_p90"][1] for r in rows)
    c1 = d["c1"]
    assert c1["round_trip_equal"] and c1["sp800_38a_f21_encrypt_ok"] and c1["sp800_38a_f22_decrypt_ok"]
    assert 0 < c1["decrypt_us_p10_p50_p90"][1] < 1e4


def test_bench_two_ranks_c5_strong_scaling():
    """C5 (BASELINE.json:11, the config of the 1/2/4/8 scaling metric) under the
    driver's --gpus N form: the 64 GiB job split into two contiguous page
    ranges, each rank checking EVERY byte of its range against the M-page
    pattern at its own offset (synth.shard; bench.plan)."""
    d = _run(["--gpus", "2", "--workload", "c5", "--extra", "none", "--steps", "2", "--warmup", "3", "--no-e2e"],
             {"KG_BENCH_SHARE_GPU": "1"}, timeout=1200)
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["comm"]["world"] == 2
    assert d["config"]["n_pages_per_gpu"] == 16777216 // 2
    assert d["check"]["pages"] == 16777216 and d["check"]["mismatched_pages"] == 0
    assert d["gpu_launches"] >= 2 * 2
    assert 0 < d["roofline"]["frac"] < 1.05
