"""Sustained (power-capped) comparison of compile-time variants of one plan: for each variant
(comma-separated ENV=VALUE list or "default"), the forward then the inverse back to back for
`seconds` each, with the NVML SM clock and power over the window; variants alternate twice.
python sustain_cmp.py <plan> <seconds> <variant> ..."""
import json
import os
import statistics
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import pynvml  # noqa: E402
import torch  # noqa: E402

import probe_plans  # noqa: E402

name, seconds = sys.argv[1], float(sys.argv[2])
variants = sys.argv[3:]
plans = []
for v in variants:
    env = {} if v == "default" else dict(kv.split("=", 1) for kv in v.split(","))
    os.environ.update(env)
    p, n, batch, dt = probe_plans.make(name, no_cubin_cache=True)
    for k in env:
        os.environ.pop(k)
    plans.append(p)
X = torch.randn(batch, n, device="cuda")
Y = torch.empty_like(X)
nb = 2 * batch * n * 4
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)


def sustain(fn):
    samples, stop = [], threading.Event()

    def sample():
        while not stop.is_set():
            samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                            pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0))
            time.sleep(0.005)
    th = threading.Thread(target=sample)
    th.start()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    n_, tot = 0, 0.0
    while tot < seconds * 1e3:
        for _ in range(50):
            fn()
        n_ += 50
        b.record()
        b.synchronize()
        tot = a.elapsed_time(b)
    stop.set()
    th.join()
    return nb / (tot / n_) / 1e6, statistics.median(s[0] for s in samples), statistics.median(s[1] for s in samples)


for rep in range(2):
    for v, p in zip(variants, plans):
        for kind, f in (("fwd", p.forward), ("inv", p.inverse)):
            gbs, mhz, w = sustain(lambda: f(X, Y))
            print(json.dumps({"plan": name, "variant": v, "rep": rep, "kind": kind, "kernel": p.kernel_name(0, dt),
                              "sustained_gbs": round(gbs, 1), "frac": round(gbs / 6454.9, 4), "sm_mhz": mhz,
                              "power_w": round(w, 1)}), flush=True)
