"""FMA-skeleton geometry sweep for one plan kernel (fwd / inv / filter): each (R, stages, warps,
pace) candidate is set through gft_plan_tuning_set / a filter rebuilt under GFT_TUNE_* env, and
timed as best of 3 x 60 back-to-back launches (the built-in tuner's 2 x 10 is within noise of
these differences).  python geo_sweep.py <cfg|rhN>[:f64][@log2batch] <fwd|inv|filt>"""
import itertools
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import workloads  # noqa: E402
from paper_1907_07875_b200 import gft  # noqa: E402

spec, kind = sys.argv[1], sys.argv[2]
spec, lb = spec.split("@") if "@" in spec else (spec, None)
name, dt = spec.split(":") if ":" in spec else (spec, "f32")
if name.startswith("rh"):
    import probe_plans
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
esz = X.element_size()


def timed(fn):
    for _ in range(10):
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


res = []
plan = new_plan(no_cubin_cache=True)
default = None
WARPS = tuple(int(w) for w in os.environ.get("SWEEP_WARPS", "4,8,12").split(","))
OBUFS = tuple(int(w) for w in os.environ.get("SWEEP_OBUF", "0").split(","))
PACES = tuple(int(w) for w in os.environ.get("SWEEP_PACE", "0,150").split(","))
RS = tuple(int(w) for w in os.environ.get("SWEEP_R", "1,2,4").split(","))
for R, S, W, pace, ob in itertools.product(RS, (2, 3), WARPS, PACES, OBUFS):
    tile = 32 * R * gn * esz
    if W * (S + ob) * tile + W * S * 8 + 1024 > 227 * 1024 or tile > 32768:
        continue
    os.environ["GFT_FMA_OBUF"] = str(ob)
    try:
        if kind == "filt":
            for k, v in (("GFT_TUNE_R", R), ("GFT_TUNE_STAGES", S), ("GFT_TUNE_WARPS", W), ("GFT_PACE_NS", pace)):
                os.environ[k] = str(v)
            f = gft.Filter(plan, np.exp(-plan.eigenvalues()), dtypes=(dt,), no_cubin_cache=True)
            frac = timed(lambda: f.apply(X, Y))
            f.close()
        else:
            k = 0 if kind == "fwd" else 1
            plan = new_plan(no_cubin_cache=True)
            plan.set_tuning({k: (R, S, W, pace)}, dt)
            fn = plan.forward if k == 0 else plan.inverse
            frac = timed(lambda: fn(X, Y))
    except gft.GFTError as e:
        continue
    res.append(((R, S, W, pace, ob), round(frac, 4)))
for k in ("GFT_TUNE_R", "GFT_TUNE_STAGES", "GFT_TUNE_WARPS", "GFT_PACE_NS", "GFT_FMA_OBUF"):
    os.environ.pop(k, None)
res.sort(key=lambda r: -r[1])
print(json.dumps({"spec": spec, "kind": kind, "top": res[:8], "n": len(res)}))
