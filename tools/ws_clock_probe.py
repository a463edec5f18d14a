"""Back-to-back cfg5b forward for ~2 s each: IO-split warp-specialised kernel vs plain pair
kernel, with NVML SM-clock / power samples during each run (is the WS kernel throttled?)."""
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
cfg = workloads.config("cfg5b")
os.environ["GFT_TC_IOSPLIT"] = "1"
ws = G.Plan.from_config(cfg, dtypes=("f32",))
os.environ.pop("GFT_TC_IOSPLIT")
pair = G.Plan.from_config(cfg, dtypes=("f32",))
X = torch.randn(cfg.batch, cfg.n, device="cuda")
Y = torch.empty_like(X)
for name, p in (("ws", ws), ("pair", pair), ("ws", ws), ("pair", pair)):
    for _ in range(5):
        p.forward(X, Y)
    torch.cuda.synchronize()
    samples, stop = [], threading.Event()

    def sample():
        while not stop.is_set():
            samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                            pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0))
            time.sleep(0.005)
    th = threading.Thread(target=sample)
    th.start()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10000):
        p.forward(X, Y)
    e.record()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    ms = s.elapsed_time(e) / 10000
    clk = sorted(c for c, _ in samples)
    pw = sorted(w for _, w in samples)
    print(json.dumps({"kernel": name, "ms": round(ms, 5), "gbs": round(2 * X.numel() * 4 / ms / 1e6),
                      "sm_mhz_median": clk[len(clk) // 2], "sm_mhz_min": clk[0],
                      "power_w_median": pw[len(pw) // 2], "samples": len(samples)}))
