"""Small launches of every kernel family for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): FMA skeleton in all three copy modes with ragged tails (packed view
cfg1, TMA tensor cfg2, 1-D bulk cfg3), fp64 (cfg4), the CTA-pair tcgen05 kernel (cfg5b), the
warp-specialised tcgen05 kernel (right-Haar 32|32), the fused filter and the host-buffer
path.  Each transform is checked by its round trip.
  compute-sanitizer --tool memcheck python tools/sanitize_driver.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_1907_07875_b200 import gft  # noqa: E402


def roundtrip(plan, rows, n, dtype):
    tdt = torch.float64 if dtype == "f64" else torch.float32
    X = torch.randn(rows, n, device="cuda", dtype=tdt)
    Y = plan.forward(X)
    Z = plan.inverse(Y)
    torch.cuda.synchronize()
    err = float((Z - X).norm() / X.norm())
    assert err < (1e-10 if dtype == "f64" else 1e-4), err
    return X


cases = [("cfg1", "f32", 4097), ("cfg2", "f32", 777), ("cfg3", "f32", 1000), ("cfg4", "f64", 513),
         ("cfg5b", "f32", 300)]
for name, dt, rows in cases:
    cfg = workloads.config(name)
    plan = gft.Plan.from_config(cfg, dtypes=(dt,))
    X = roundtrip(plan, rows, cfg.n, dt)
    if name == "cfg2":
        filt = gft.Filter(plan, np.exp(-plan.eigenvalues()), dtypes=(dt,))
        filt.apply(X)
        Xh = X.cpu().pin_memory()
        Yh = torch.empty_like(Xh).pin_memory()
        ws = torch.empty(4 * 256 * cfg.n * 2, device="cuda")
        plan.execute_host(0, Xh, Yh, ws, 256)
        torch.cuda.synchronize()
        filt.close()
    print(name, plan.kernel_name(0, dt), "ok", flush=True)
    plan.close()
n, s_, d_, w_, loops, norm = workloads.right_haar_bench_graph(workloads.RIGHT_HAAR_BENCH_CASES[0])
plan = gft.Plan(n, s_, d_, w_, loops, dtypes=("f32",), normalized=norm)
roundtrip(plan, 1000, n, "f32")
print("rh0", plan.kernel_name(0, "f32"), "ok", flush=True)
plan.close()
