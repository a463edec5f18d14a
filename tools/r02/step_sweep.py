"""Geometry of cfg5a's forward / inverse kernels chosen inside the headline step (bench.py:
5a fwd, 5b fwd, 5a inv, 5b inv back to back), not in isolation -- the isolated back-to-back
sweeps disagree with the step (cfg5a fwd with 2,2,3,150,2: 0.84 of HBM when launched after
itself, fast after another kernel).  Each argument is "fwd=R,S,W,pace,obuf;inv=R,S,W,pace,obuf"
(either part optional, "default" = tuning.tsv); candidates are timed in interleaved rounds
(best of 3 x 20 steps per round, 3 rounds); prints the median step time and the 5a share.
NOTE (r44-r48): with many candidates the GPU is at the power cap from the second round on, so
the medians are SUSTAINED-regime numbers (default 0.527 ms here vs 0.4986 ms for bench.py's
burst on the same box); step_sweep2.py measures both regimes per candidate."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_1907_07875_b200 import gft  # noqa: E402

ca, cb = workloads.config("cfg5a"), workloads.config("cfg5b")
pb = gft.Plan.from_config(cb, dtypes=("f32",))
XA = workloads.signals(ca, dtype="f32").cuda()
XB = workloads.signals(cb, dtype="f32").cuda()
YA, ZA, YB, ZB = (torch.empty_like(t) for t in (XA, XA, XB, XB))


def make(spec):
    parts = {} if spec == "default" else dict(p.split("=") for p in spec.split(";"))
    plans = {}
    for kind, key in ((0, "fwd"), (1, "inv")):
        if key in parts:
            R, S, W, pace, ob = (int(v) for v in parts[key].split(","))
            os.environ["GFT_FMA_OBUF"] = str(ob)
            p = gft.Plan.from_config(ca, dtypes=("f32",), no_cubin_cache=True)
            p.set_tuning({kind: (R, S, W, pace)}, "f32")
            os.environ.pop("GFT_FMA_OBUF")
        else:
            p = gft.Plan.from_config(ca, dtypes=("f32",))
        plans[kind] = p
    return plans


cands = sys.argv[1:] or ["default"]
made = [(c, make(c)) for c in cands]
# every candidate computes the same rows bit for bit (same FFMA order per row)
ref_y = made[0][1][0].forward(XA)
ref_z = made[0][1][1].inverse(ref_y)
for c, pl in made[1:]:
    y = pl[0].forward(XA)
    assert torch.equal(y, ref_y), c
    assert torch.equal(pl[1].inverse(y), ref_z), c
del ref_y, ref_z


def timed(pl):
    def step():
        pl[0].forward(XA, YA)
        pb.forward(XB, YB)
        pl[1].inverse(YA, ZA)
        pb.inverse(YB, ZB)
    for _ in range(5):
        step()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20):
            step()
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b) / 20)
    return best


def copy_step_ms():
    """the same bytes as plain device copies (what this box moves for pure data movement)"""
    def step():
        YA.copy_(XA); YB.copy_(XB); ZA.copy_(YA); ZB.copy_(YB)
    for _ in range(5):
        step()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20):
            step()
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b) / 20)
    return best


print(json.dumps({"copy_step_ms": round(copy_step_ms(), 5)}), flush=True)
res = {c: [] for c in cands}
for _ in range(3):
    for c, pl in made:
        res[c].append(timed(pl))
for c, pl in made:
    ms = statistics.median(res[c])
    print(json.dumps({"cand": c, "step_ms": round(ms, 5), "signals_per_s": round(2 * (1 << 20) / (ms * 1e-3)),
                      "fwd": pl[0].kernel_name(0, "f32"), "inv": pl[1].kernel_name(1, "f32")}), flush=True)
