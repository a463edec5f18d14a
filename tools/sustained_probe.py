"""Sustained (power-capped) vs burst throughput: each kernel back to back for ~2 s with NVML
SM-clock / power samples, next to a 20-launch burst.  cfg5b is run through both tensor-core
kernels (plain CTA pair, and the opt-in IO-split warp-specialised one).
  python tools/sustained_probe.py  ->  one JSON line per kernel"""
import json
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import pynvml  # noqa: E402
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_1907_07875_b200 import gft as G  # noqa: E402

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)


def run(label, plan, cfg, seconds=2.0):
    X = torch.randn(cfg.batch, cfg.n, device="cuda")
    Y = torch.empty_like(X)
    nb = 2 * X.numel() * 4

    def timed(iters):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(iters):
            plan.forward(X, Y)
        e.record()
        torch.cuda.synchronize()
        return s.elapsed_time(e) / iters
    for _ in range(5):
        plan.forward(X, Y)
    torch.cuda.synchronize()
    time.sleep(1.0)                       # let the clocks recover between kernels
    burst = timed(20)
    iters = int(seconds / (burst * 1e-3))
    samples, stop = [], threading.Event()

    def sample():
        while not stop.is_set():
            samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                            pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0))
            time.sleep(0.005)
    th = threading.Thread(target=sample)
    th.start()
    sus = timed(iters)
    stop.set()
    th.join()
    clk = sorted(c for c, _ in samples)
    pw = sorted(w for _, w in samples)
    print(json.dumps({"plan": label, "kernel": plan.kernel_name(0, "f32"),
                      "burst_gbs": round(nb / burst / 1e6), "sustained_gbs": round(nb / sus / 1e6),
                      "sustained_sm_mhz_median": clk[len(clk) // 2], "power_w_median": pw[len(pw) // 2],
                      "launches": iters}), flush=True)


if __name__ == "__main__":
    names = sys.argv[1:] or ["cfg2", "cfg5a", "cfg5b"]
    for name in names:
        cfg = workloads.config(name)
        run(name + (" suspend=%s" % os.environ["GFT_SUSPEND_NS"] if "GFT_SUSPEND_NS" in os.environ else ""),
            G.Plan.from_config(cfg, dtypes=("f32",)), cfg)
    if not sys.argv[1:]:
        cfg = workloads.config("cfg5b")
        os.environ["GFT_TC_IOSPLIT"] = "1"
        run("cfg5b io-split WS", G.Plan.from_config(cfg, dtypes=("f32",)), cfg)
