"""Kernels for the r02 ncu comparison of fused filters vs plain transforms (FMA skeleton):
cfg4 f64 and cfg5a forward + heat-kernel filter, and the right-Haar 32|32 tcgen05 forward;
each launched 3 times back to back (profile the 2nd)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import probe_plans  # noqa: E402
import workloads  # noqa: E402
from paper_1907_07875_b200 import gft  # noqa: E402

for name, dt in (("cfg4", "f64"), ("cfg5a", "f32")):
    cfg = workloads.config(name)
    p = gft.Plan.from_config(cfg, dtypes=(dt,))
    f = gft.Filter(p, np.exp(-p.eigenvalues()), dtypes=(dt,))
    X = torch.randn(cfg.batch, cfg.n, device="cuda", dtype=torch.float64 if dt == "f64" else torch.float32)
    Y = torch.empty_like(X)
    for fn in (lambda: p.forward(X, Y), lambda: f.apply(X, Y)):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
p, n, batch, dt = probe_plans.make("rh0")
X = torch.randn(batch, n, device="cuda")
Y = torch.empty_like(X)
for _ in range(3):
    p.forward(X, Y)
torch.cuda.synchronize()
