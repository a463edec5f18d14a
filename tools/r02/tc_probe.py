"""tcgen05 kernel probe: cfg5b forward / inverse burst (20 launches) and sustained (~2 s back
to back at the power cap) GB/s with the median SM clock, for the kernel variant the current
environment selects (GFT_TC_* knobs; compiled with NVRTC).  Optional argv[1]: config name."""
import json
import os
import statistics
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import workloads  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import probe_plans  # noqa: E402
from paper_1907_07875_b200 import gft  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg5b"
secs = float(sys.argv[2]) if len(sys.argv) > 2 else 2.0
p, n, batch, _ = probe_plans.make(name, no_cubin_cache=True)
X = torch.randn(batch, n, device="cuda")
Y = torch.empty_like(X)
Z = torch.empty_like(X)
nb = 2 * batch * n * 4
out = {"env": {k: v for k, v in os.environ.items() if k.startswith("GFT_")}, "cfg": name,
       "fwd": p.kernel_name(0, "f32"), "inv": p.kernel_name(1, "f32")}
# parity vs fp64 dense basis
U = torch.from_numpy(p.basis()).cuda()
p.forward(X, Y)
ref = X.double() @ U
out["fwd_err"] = float(((Y.double() - ref).norm(dim=1) / ref.norm(dim=1)).max())
p.inverse(Y, Z)
out["rt_err"] = float(((Z.double() - X.double()).norm(dim=1) / X.double().norm(dim=1)).max())

import pynvml  # noqa: E402
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
samples, stop = [], threading.Event()


def sampler():
    while not stop.is_set():
        samples.append((time.perf_counter(), pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                        pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0))
        time.sleep(0.005)


th = threading.Thread(target=sampler, daemon=True)
th.start()


def timed(fn, iters):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / iters


fns = (("fwd", lambda: p.forward(X, Y)), ("inv", lambda: p.inverse(Y, Z)))
for tag, fn in fns:   # cold bursts first (after an idle pause: a hot GPU sits at a capped clock)
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    time.sleep(4.0)
    ms = timed(fn, 20)
    out[tag + "_burst_gbs"] = round(nb / ms / 1e6, 1)
for tag, fn in (fns if secs > 0 else ()):
    t0 = time.perf_counter()
    ms = timed(fn, 20)
    n_it = max(1, int(secs * 1e3 / ms))
    ms = timed(fn, n_it)
    t1 = time.perf_counter()
    w = [s for s in samples if t0 + 0.5 * (t1 - t0) <= s[0] <= t1]
    out[tag + "_sustained_gbs"] = round(nb / ms / 1e6, 1)
    out[tag + "_sustained_mhz"] = statistics.median([s[1] for s in w]) if w else None
    out[tag + "_sustained_w"] = round(statistics.median([s[2] for s in w]), 1) if w else None
stop.set()
print(json.dumps(out))
