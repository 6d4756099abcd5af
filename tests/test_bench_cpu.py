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
