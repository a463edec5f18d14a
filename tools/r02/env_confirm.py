"""Compare compile-time variants of one plan: each argument is a comma-separated list of
ENV=VALUE settings (or "default") under which the plan is generated; forward and inverse of
every variant are timed in interleaved rounds (best of 3 x 40 back-to-back launches per round,
3 rounds); prints median GB/s and the fraction of the 6455 GB/s copy peak per variant.
python env_confirm.py <plan: cfgN | rhN> <variant> ..."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch  # noqa: E402

import probe_plans  # noqa: E402
from paper_1907_07875_b200 import gft  # noqa: E402

name = sys.argv[1]
variants = sys.argv[2:]
plans = []
for v in variants:
    env = {} if v == "default" else dict(kv.split("=", 1) for kv in v.split(","))
    os.environ.update(env)
    p, n, batch, dt = probe_plans.make(name, no_cubin_cache=True)
    for k in env:
        os.environ.pop(k)
    plans.append(p)
X = torch.randn(batch, n, device="cuda", dtype=torch.float64 if dt == "f64" else torch.float32)
Y = torch.empty_like(X)
nb = 2 * batch * n * X.element_size()


def timed(fn):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(40):
            fn()
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b) / 40)
    return nb / best / 1e6


# ENV_CONFIRM_FILTER=1: the "inv" column times the heat-kernel fused filter instead
filters = []
if os.environ.get("ENV_CONFIRM_FILTER") == "1":
    import numpy as np
    for v, p in zip(variants, plans):
        env = {} if v == "default" else dict(kv.split("=", 1) for kv in v.split(","))
        os.environ.update(env)
        filters.append(gft.Filter(p, np.exp(-p.eigenvalues()), dtypes=(dt,), no_cubin_cache=True))
        for k in env:
            os.environ.pop(k)
res = {(v, k): [] for v in variants for k in ("fwd", "inv")}
for _ in range(3):
    for j, (v, p) in enumerate(zip(variants, plans)):
        res[(v, "fwd")].append(timed(lambda: p.forward(X, Y)))
        if filters:
            res[(v, "inv")].append(timed(lambda: filters[j].apply(X, Y)))
        else:
            res[(v, "inv")].append(timed(lambda: p.inverse(X, Y)))
for v, p in zip(variants, plans):
    f, i = statistics.median(res[(v, "fwd")]), statistics.median(res[(v, "inv")])
    print(json.dumps({"plan": name, "variant": v, "kernel": p.kernel_name(0, dt), "fwd_gbs": round(f, 1),
                      "inv_gbs": round(i, 1), "fwd_frac": round(f / 6454.9, 4), "inv_frac": round(i / 6454.9, 4)}),
          flush=True)
