"""One config's forward + inverse pair (X -> Y -> Z, back to back) in BOTH regimes per geometry:
burst (idle pause, 5 warm-up, 20 timed pairs) and sustained (1.5 s of pairs, then the mean of the
next 3 x 200 pairs at the power cap).  python regime_sweep.py <cfg> <f32|f64> cand...  with cand =
"default" | "copy" | "R,S,W,pace,obuf" (both directions).  Interleaved rounds, medians; GB/s =
algorithmic bytes of the pair / time, and the fraction of the copy pair measured the same way.
SWEEP_FILTER=1: the fused filter (X -> Y, then Y -> Z) instead of the forward / inverse pair, the
geometry set through the GFT_TUNE_* / GFT_PACE_NS / GFT_FMA_OBUF knobs at kernel generation."""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_1907_07875_b200 import gft  # noqa: E402

name, dt = sys.argv[1], sys.argv[2]
batch = int(os.environ.get("SWEEP_BATCH", "0")) or None
cfg = workloads.config(name)
X = workloads.signals(cfg, batch=batch, dtype=dt).cuda()
Y, Z = torch.empty_like(X), torch.empty_like(X)
nbytes = 2 * 2 * X.numel() * X.element_size()
stream = torch.cuda.current_stream()


FILTER = os.environ.get("SWEEP_FILTER") == "1"
MODE = os.environ.get("SWEEP_MODE", "pair")   # pair | fwd | inv (forward-only / inverse-only streams)


def make_filter(spec):
    import numpy as np
    keys = ("GFT_TUNE_R", "GFT_TUNE_STAGES", "GFT_TUNE_WARPS", "GFT_PACE_NS", "GFT_FMA_OBUF")
    if spec != "default":
        for k, v in zip(keys, spec.split(",")):
            os.environ[k] = v
    p = gft.Plan.from_config(cfg, dtypes=(dt,))
    f = gft.Filter(p, np.exp(-0.5 * p.eigenvalues()), dtypes=(dt,), no_cubin_cache=spec != "default")
    for k in keys:
        os.environ.pop(k, None)
    return f


def make(spec):
    if spec == "copy":
        return None
    if FILTER:
        return make_filter(spec)
    if spec == "default":
        return gft.Plan.from_config(cfg, dtypes=(dt,))
    R, S, W, pace, ob = (int(v) for v in spec.split(","))
    os.environ["GFT_FMA_OBUF"] = str(ob)
    p = gft.Plan.from_config(cfg, dtypes=(dt,), no_cubin_cache=True)
    p.set_tuning({0: (R, S, W, pace), 1: (R, S, W, pace)}, dt)
    os.environ.pop("GFT_FMA_OBUF")
    return p


def stepper(p):
    if p is None:
        def step():
            Y.copy_(X); Z.copy_(Y)
        return step

    if FILTER:
        def step():
            p.apply(X, Y, stream)
            p.apply(Y, Z, stream)
        return step

    if MODE == "fwd":      # forward-only stream (two launches per step, like the pair)
        def step():
            p.forward(X, Y, stream)
            p.forward(X, Z, stream)
        return step
    if MODE == "inv":
        def step():
            p.inverse(X, Y, stream)
            p.inverse(X, Z, stream)
        return step

    def step():
        p.forward(X, Y, stream)
        p.inverse(Y, Z, stream)
    return step


def timed(step, n):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        step()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / n


def burst(step):
    torch.cuda.synchronize()
    time.sleep(1.5)
    for _ in range(5):
        step()
    torch.cuda.synchronize()
    return timed(step, 20)


def sustained(step):
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < 1.5:
        timed(step, 200)
    return statistics.mean(timed(step, 200) for _ in range(3))


cands = sys.argv[3:] or ["copy", "default"]
made = []
for c in cands:
    try:
        made.append((c, make(c)))
    except gft.GFTError as e:   # geometry not realisable for this kernel: skip
        print(json.dumps({"cand": c, "skipped": str(e)[:80]}), flush=True)
cands = [c for c, _ in made]
res = {c: ([], []) for c in cands}
for _ in range(3):
    for c, p in made:
        st = stepper(p)
        res[c][0].append(burst(st))
        res[c][1].append(sustained(st))
cb = statistics.median(res["copy"][0]) if "copy" in res else None
cs = statistics.median(res["copy"][1]) if "copy" in res else None
for c, p in made:
    b, s = statistics.median(res[c][0]), statistics.median(res[c][1])
    print(json.dumps({"cfg": name + ("_filter" if FILTER else "") + ("" if MODE == "pair" else "_" + MODE), "dtype": dt, "cand": c, "burst_gbs": round(nbytes / b / 1e6, 1),
                      "sustained_gbs": round(nbytes / s / 1e6, 1),
                      "burst_vs_copy": round(cb / b, 4) if cb else None,
                      "sustained_vs_copy": round(cs / s, 4) if cs else None}), flush=True)
