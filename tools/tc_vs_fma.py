"""Where do tcgen05 leaves beat CUDA-core FMA leaves?  Times the same plan both ways
(forward, fp32, 2^20 device-resident signals) on graphs whose leaves are 32..64 wide.

  python tools/tc_vs_fma.py  ->  one JSON line per plan
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_1907_07875_b200 import gft as G  # noqa: E402


def timed(fn, iters=30):
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


def graphs():
    rng = np.random.default_rng(1)
    for a, b in ((32, 32), (40, 40), (48, 48), (64, 64), (24, 40)):
        s, d, w, loops, _ = workloads.random_bipartite_graph(rng, a, b, density=0.3)
        yield "norm-bip %d|%d" % (a, b), (a + b, s, d, w, loops, None), {"normalized": True}
    for n in (64, 96, 128):
        s, d, w, loops, phi = workloads.random_symmetric_graph(rng, n, density=0.3, fixed_frac=0.0)
        yield "sym-random %d" % n, (n, s, d, w, loops, phi), {}


def main():
    for label, (n, s, d, w, loops, phi), kw in graphs():
        X = torch.randn(1 << 20, n, device="cuda")
        Y = torch.empty_like(X)
        row = {"graph": label, "n": n}
        for tag, no_tc in (("tc", False), ("fma", True)):
            plan = G.Plan(n, s, d, w, loops, phi, dtypes=("f32",), no_tensor_cores=no_tc, **kw)
            row["leaves"] = plan.leaf_sizes()
            row["sum_k2"] = plan.info()["sum_k2"]
            ms = timed(lambda: plan.forward(X, Y))
            row[tag] = {"ms": round(ms, 5), "gbs": round(2 * X.numel() * 4 / ms / 1e6, 1),
                        "kernel": plan.kernel_name(0, "f32")}
            plan.close()
        row["fma_over_tc"] = round(row["tc"]["ms"] / row["fma"]["ms"], 3)
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
