"""Headline-step sweep of cfg5a's forward / inverse geometry in BOTH regimes per candidate:
burst  = after an idle pause (clock back at its maximum): 5 warm-up + 20 timed steps, as
         bench.py's timed region;
sustained = 1.5 s of back-to-back steps, then the mean step time of the next ~0.7 s (the
         1000 W power cap holds the SM clock near 1.5-1.6 GHz), as bench.py's sustained arm.
Candidates as in step_sweep.py ("fwd=R,S,W,pace,obuf;inv=..." or "default"); the copy step
(the same bytes as plain torch copies) is measured the same way.  Rounds are interleaved;
medians are printed."""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_1907_07875_b200 import gft  # noqa: E402

ROUNDS = int(os.environ.get("SWEEP_ROUNDS", "3"))
ca, cb = workloads.config("cfg5a"), workloads.config("cfg5b")
pb = gft.Plan.from_config(cb, dtypes=("f32",))
XA = workloads.signals(ca, dtype="f32").cuda()
XB = workloads.signals(cb, dtype="f32").cuda()
YA, YB = torch.empty_like(XA), torch.empty_like(XB)     # bench.py's allocation order
ZA, ZB = torch.empty_like(XA), torch.empty_like(XB)
stream = torch.cuda.current_stream()


def make(spec):
    parts = {} if spec in ("default", "copy") else dict(p.split("=") for p in spec.split(";"))
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


def stepper(spec, pl):
    if spec == "copy":
        def step():
            YA.copy_(XA); YB.copy_(XB); ZA.copy_(YA); ZB.copy_(YB)
        return step

    def step():
        pl[0].forward(XA, YA, stream)
        pb.forward(XB, YB, stream)
        pl[1].inverse(YA, ZA, stream)
        pb.inverse(YB, ZB, stream)
    return step


def timed_steps(step, n):
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
    return timed_steps(step, 20)


def sustained(step):
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < 1.5:
        timed_steps(step, 200)
    return statistics.mean(timed_steps(step, 400) for _ in range(3))


cands = sys.argv[1:] or ["default"]
made = [(c, make(c)) for c in cands]
ref_y = made[0][1][0].forward(XA)
ref_z = made[0][1][1].inverse(ref_y)
for c, pl in made[1:]:
    if c == "copy":
        continue
    y = pl[0].forward(XA)
    assert torch.equal(y, ref_y), c
    assert torch.equal(pl[1].inverse(y), ref_z), c
    del y
del ref_y, ref_z
res = {c: ([], []) for c in cands}
for _ in range(ROUNDS):
    for c, pl in made:
        st = stepper(c, pl)
        res[c][0].append(burst(st))
        res[c][1].append(sustained(st))
for c, pl in made:
    b, s = statistics.median(res[c][0]), statistics.median(res[c][1])
    print(json.dumps({"cand": c, "burst_ms": round(b, 5), "sustained_ms": round(s, 5),
                      "burst_all": [round(v, 4) for v in res[c][0]], "sustained_all": [round(v, 4) for v in res[c][1]],
                      "fwd": None if c == "copy" else pl[0].kernel_name(0, "f32")[-8:],
                      "inv": None if c == "copy" else pl[1].kernel_name(1, "f32")[-8:]}), flush=True)
