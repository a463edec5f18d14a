"""bench.py contract checks that run without a GPU (the reference arm is the CPU oracle)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--steps", "2", "--warmup", "3", "--ref-rows", "20000"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "config", "cpu_baseline", "e2e", "dtype"):
        assert k in d, k
    assert d["value"] > 0 and d["unit"] == "signals/s"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["config"]["workload"].startswith("cfg5 mixed")
    assert len(lines[0].encode()) <= 2048


def test_headline_line_compaction():
    """The headline keeps every contract key and stays under the limit: floats are rounded
    first, and only then are the least important keys dropped, in a fixed order."""
    import bench
    out = {"metric": "m", "value": 4212569599.193279, "unit": "signals/s", "ms_per_step": 0.4978320121765137,
           "roofline": {"frac": 1.0143000001, "achieved": 6544.41234567}, "peaks_tflops": {"a": 1.23456789},
           "cpu_baseline": {"value": 4.7e6, "sample": "x" * 300}, "e2e": {"value": 59690925.760148704},
           "kernels": {"share": {"a": 0.1}, "fast_vs_best_dense": 1.1234567}}
    line = bench.headline_line(dict(out))
    d = json.loads(line)
    assert d["value"] == out["value"] and d["ms_per_step"] == out["ms_per_step"]
    assert d["roofline"]["frac"] == 1.0143 and d["e2e"]["value"] == 59690900.0
    assert "kernels" in d and "peaks_tflops" in d
    small = bench.headline_line(dict(out), limit=len(line) - 1)
    assert "peaks_tflops" not in json.loads(small) and "kernels" in json.loads(small)
    tiny = json.loads(bench.headline_line(dict(out), limit=100))
    for k in ("metric", "value", "unit", "roofline", "e2e", "cpu_baseline"):
        assert k in tiny
    assert "kernels" not in tiny and "sample" not in tiny["cpu_baseline"]
