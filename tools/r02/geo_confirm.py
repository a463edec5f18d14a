"""Confirm geometry candidates of the CUDA-core kernels: each (R, stages, warps, pace, obuf)
candidate of a (config, kind) is built once, then all are timed in interleaved rounds (best of
3 x 60 back-to-back launches per round, 3 rounds); prints the median fraction of the measured
copy peak per candidate.  python geo_confirm.py <cfg|rhN>[:f64][@log2batch] <fwd|inv|filt> R,S,W,pace,obuf ..."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_1907_07875_b200 import gft  # noqa: E402

spec, kind = sys.argv[1], sys.argv[2]
cands = [tuple(int(v) for v in c.split(",")) for c in sys.argv[3:]]
spec_, lb = spec.split("@") if "@" in spec else (spec, None)
name, dt = spec_.split(":") if ":" in spec_ else (spec_, "f32")
if name.startswith("rh"):   # right-Haar bench plans (workloads.RIGHT_HAAR_BENCH_CASES), 2^20 signals
    case = workloads.RIGHT_HAAR_BENCH_CASES[int(name[2:])]
    dt = case[4]
    gn, gs, gd, gw, gl, gnorm = workloads.right_haar_bench_graph(case)
    NB = 1 << 20

    def new_plan(**kw):
        return gft.Plan(gn, gs, gd, gw, gl, dtypes=(dt,), normalized=gnorm, **kw)
else:
    cfg = workloads.config(name)
    gn, NB = cfg.n, cfg.batch

    def new_plan(**kw):
        return gft.Plan.from_config(cfg, dtypes=(dt,), **kw)
if lb:
    NB = 1 << int(lb)
tdt = torch.float64 if dt == "f64" else torch.float32
X = torch.randn(NB, gn, device="cuda", dtype=tdt)
Y = torch.empty_like(X)
nb = 2 * NB * gn * X.element_size()
fns = []
for c in [None] + cands:
    if c is not None:
        R, S, W, pace, ob = c
        os.environ.update(GFT_TUNE_R=str(R), GFT_TUNE_STAGES=str(S), GFT_TUNE_WARPS=str(W), GFT_PACE_NS=str(pace),
                          GFT_FMA_OBUF=str(ob))
    p = new_plan(no_cubin_cache=True)
    f = gft.Filter(p, np.exp(-p.eigenvalues()), dtypes=(dt,), no_cubin_cache=True) if kind == "filt" else None
    for k in ("GFT_TUNE_R", "GFT_TUNE_STAGES", "GFT_TUNE_WARPS", "GFT_PACE_NS", "GFT_FMA_OBUF"):
        os.environ.pop(k, None)
    fn = {"fwd": (lambda p=p: p.forward(X, Y)), "inv": (lambda p=p: p.inverse(X, Y)),
          "filt": (lambda f=f: f.apply(X, Y))}[kind]
    fns.append(("default" if c is None else ",".join(map(str, c)), fn, p, f))


def timed(fn):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(60):
            fn()
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b) / 60)
    return nb / best / 1e6 / 6454.9


res = {tag: [] for tag, *_ in fns}
for _ in range(3):
    for tag, fn, _p, _f in fns:
        res[tag].append(timed(fn))
print(json.dumps({"spec": spec, "kind": kind, "median": {t: round(statistics.median(v), 4) for t, v in res.items()},
                  "min": {t: round(min(v), 4) for t, v in res.items()}}))
