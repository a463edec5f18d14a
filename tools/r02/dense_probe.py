"""Dense comparison GEMM geometry probe: time the CUDA-core dense kernels of cfg5b / cfg5a /
cfg4 (f32, f64) under GFT_DG_TM / GFT_DG_TN / GFT_DG_THREADS overrides (set per process)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_1907_07875_b200 import gft  # noqa: E402

PEAK = {"f32": 73.4e12, "f64": 33.9e12}
out = {"env": {k: v for k, v in os.environ.items() if k.startswith("GFT_DG")}}
for name, dt in (("cfg5b", "f32"), ("cfg5a", "f32"), ("cfg4", "f32"), ("cfg4", "f64")):
    cfg = workloads.config(name)
    p = gft.Plan.from_config(cfg, dtypes=(dt,), no_cubin_cache=True)
    tdt = torch.float64 if dt == "f64" else torch.float32
    X = torch.randn(cfg.batch, cfg.n, device="cuda", dtype=tdt)
    Y = torch.empty_like(X)
    for _ in range(3):
        p.dense_forward(X, Y)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10):
        p.dense_forward(X, Y)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 10
    U = torch.from_numpy(p.basis()).to(device="cuda", dtype=tdt)
    err = float(((Y - X @ U).norm(dim=1) / (X @ U).norm(dim=1)).max())
    out["%s_%s" % (name, dt)] = {"ms": round(ms, 4), "frac": round(2.0 * cfg.n ** 2 * cfg.batch / (ms * 1e-3) / PEAK[dt], 4),
                                 "kernel": p.kernel_name(2, dt), "err": err}
print(json.dumps(out))
