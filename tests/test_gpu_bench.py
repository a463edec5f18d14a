"""The bench contract on the GPU, run with the driver's exact command line: the LAST stdout
line parses, is at most 2 KiB (the driver keeps a bounded stdout tail), carries every key the
driver reads (metric / value / unit / n_gpus / steps / warmup / ms_per_step / roofline /
cpu_baseline / e2e / gpu_launches / clocks ...) and its numbers are self-consistent."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_driver_command():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "1", "--steps", "20",
                          "--warmup", "5"], capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    last = out.stdout.rstrip("\n").splitlines()[-1]
    assert len(last.encode()) <= 2048, len(last.encode())
    d = json.loads(last)
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e",
              "gpu_launches", "clocks", "sustained"):
        assert k in d, k
    assert d["steps"] == 20 and d["warmup"] == 5 and d["n_gpus"] == 1 and d["higher_is_better"] is True
    assert "cfg5 mixed" in d["config"]["workload"]
    B = d["config"]["global_batch"]
    assert B == 2 << 20
    assert abs(d["value"] - B / (d["ms_per_step"] * 1e-3)) / d["value"] < 1e-6
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0.5 < r["frac"] < 1.2
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3
    assert "n128" in r["kernel"]   # the dominant kernel is cfg5b's
    assert d["gpu_launches"] == 4 * d["steps"]
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert e["roundtrip_max_rel_err"] < 1e-5
    c = d["cpu_baseline"]
    assert c["kind"] == "oracle" and c["cores"] >= 1 and c["value"] > 0
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]
    s = d["sustained"]
    assert s["seconds"] >= 2.0 and s["value"] > 0
    assert s["dense_tc"]["ms_per_step"] > 0 and s["dense_tc"]["fast_speedup"] > 0
    assert s["copy"]["ms_per_step"] > 0 and 0.5 < s["copy"]["fast_frac_of_copy"] < 1.5
    k = d["kernels"]   # the in-run dense comparisons must survive the size limit
    assert set(k["dense_ms_per_step"]) == {"fma", "tc", "cublas"} and k["fast_vs_best_dense"] > 0
