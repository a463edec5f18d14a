"""Skeleton ceiling: an edgeless graph of n nodes plans to n 1x1 leaves (identity GFT), so its
kernel is the pure load/store skeleton.  Compares it (back to back) with the real plan of a
config and a torch device copy of the same bytes.   python tools/skeleton_ceiling.py cfg3"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_1907_07875_b200 import gft as G  # noqa: E402


def b2b(fn, iters=30):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


for name in sys.argv[1:] or ["cfg3"]:
    cfg = workloads.config(name)
    dt = cfg.dtypes[0]
    tdt = torch.float64 if dt == "f64" else torch.float32
    X = torch.randn(cfg.batch, cfg.n, device="cuda", dtype=tdt)
    Y = torch.empty_like(X)
    nb = 2 * X.numel() * X.element_size()
    real = G.Plan.from_config(cfg, dtypes=(dt,))
    ident = G.Plan(cfg.n, np.zeros(0, np.int32), np.zeros(0, np.int32), np.zeros(0), dtypes=(dt,))
    out = {"config": name,
           "real_gbs": nb / b2b(lambda: real.forward(X, Y)) / 1e6,
           "identity_skeleton_gbs": nb / b2b(lambda: ident.forward(X, Y)) / 1e6,
           "torch_copy_gbs": nb / b2b(lambda: Y.copy_(X)) / 1e6,
           "identity_kernel": ident.kernel_name(0, dt)}
    print(json.dumps(out))
