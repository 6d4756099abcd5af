"""bench.py contract pieces that run without a GPU: the reference arm (the
oracle on the host cores) prints one JSON line with the required keys."""
import json
import os
import subprocess
import sys

from conftest import ROOT


def test_reference_arm_json_line():
    env = dict(os.environ, PYTHONPATH=ROOT)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "2",
                          "--warmup", "3", "--ref-step-seconds", "0.2"],
                         capture_output=True, text=True, timeout=300, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["unit"] == "GB/s" and d["value"] > 0
    assert d["steps"] == 2 and d["warmup"] == 3 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert "workload" in d["config"]


def test_compute_peak_formula():
    sys.path.insert(0, ROOT)
    import bench
    # 148 SMs x 1965 MHz x 32 lookups/clk / 160 lookups per 16 B block (AES-128)
    assert abs(bench.compute_peak_gbs(16, 1965.0) - 930.624) < 1e-6
    assert abs(bench.compute_peak_gbs(32, 1965.0) - 664.7314285714286) < 1e-6


def test_load_peaks_tolerates_key_names(tmp_path, monkeypatch):
    """MEASURED_PEAKS.json is driver-written: bench.py reads the HBM copy
    bandwidth and the max SM clock whatever the exact key names, and falls
    back (never crashes) when it cannot find them."""
    sys.path.insert(0, ROOT)
    import bench
    monkeypatch.setattr(bench, "ROOT", str(tmp_path))
    assert bench.load_peaks()["_fallback"] is True                       # no file
    (tmp_path / "MEASURED_PEAKS.json").write_text(json.dumps({"hbm_copy_gbs": 6545.9, "sm_clock_max_mhz": 1965}))
    p = bench.load_peaks()
    assert p["hbm_gbs"] == 6545.9 and p["sm_max_mhz"] == 1965.0 and "_fallback" not in p
    (tmp_path / "MEASURED_PEAKS.json").write_text("{not json")
    assert bench.load_peaks()["_fallback"] is True
    (tmp_path / "MEASURED_PEAKS.json").write_text(json.dumps({"something": 1}))
    assert bench.load_peaks()["_fallback"] is True


def test_csv_rows_from_a_line():
    """--csv: the line's numbers as SURVEY.md §5 rows (one per config x residency,
    one per sweep point x path), computed from the JSON line alone."""
    sys.path.insert(0, ROOT)
    import bench
    roof = {"peak": 930.624, "frac": 0.9}
    line = {"n_gpus": 1, "config": {"name": "c2", "dir": "decrypt", "key_bits": 128, "n_pages_per_gpu": 65536},
            "value": 837.5616, "ms_per_step": 0.3205, "roofline": roof, "clocks": {"sm_mhz": 1965, "sm_max_mhz": 1965},
            "e2e": {"value": 48.0, "step_ms_min_median_max": [5.4, 5.5, 5.6],
                    "link_duplex_aggregate_gbs_per_direction": 50.0},
            "cpu_baseline": {"cores": 16},
            "configs": {"c3": {"dir": "encrypt", "key_bits": 256, "n_pages_per_gpu": 262144, "value": 600.0,
                               "ms_per_step": 1.79, "roofline": {"peak": 664.73, "frac": 0.9026}, "e2e": None}},
            "c4_sweep": {"oracle_threads": 16,
                         "rows": [{"pages": 1, "hbm_us": 16.384, "pinned_us": 20.0, "oracle_T_us": 2000.0}]}}
    rows = bench.csv_rows(line)
    assert [tuple(r[k] for k in ("config", "residency")) for r in rows] == [
        ("c2", "hbm"), ("c2", "pinned"), ("c3", "hbm"), ("c4", "hbm"), ("c4", "pinned"), ("c4", "oracle_threads")]
    assert all(set(r) == set(bench.CSV_COLUMNS) for r in rows)
    assert rows[0]["gbps"] == 837.562 and rows[0]["pct_roofline"] == 90.0 and rows[0]["latency_us_p50"] == 320.5
    assert rows[1]["pct_roofline"] == 96.0 and rows[1]["roofline_gbps"] == 50.0
    assert rows[2]["key_bits"] == 256 and rows[2]["n_pages"] == 262144
    assert rows[3]["gbps"] == 0.25 and rows[4]["roofline_gbps"] == 50.0        # 4096 B / 16.384 us; pinned vs the link
    assert rows[5]["host_cores"] == 16 and rows[5]["roofline_gbps"] == ""
