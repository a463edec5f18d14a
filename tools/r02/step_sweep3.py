"""Brute-force burst sweep of cfg5a's forward (or inverse) geometry INSIDE the headline step:
R x stages x warps x pace x obuf, each candidate compiled (thread pool), checked bit-identical
to the default, timed as bench.py times (idle pause, 5 warm-up + 20 steps), 2 interleaved
rounds, best-of; prints every candidate sorted by step time.  python step_sweep3.py fwd|inv"""
import concurrent.futures as cf
import itertools
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_1907_07875_b200 import gft  # noqa: E402

which = sys.argv[1]
kind = 0 if which == "fwd" else 1
ca, cb = workloads.config("cfg5a"), workloads.config("cfg5b")
pb = gft.Plan.from_config(cb, dtypes=("f32",))
pa = gft.Plan.from_config(ca, dtypes=("f32",))
XA = workloads.signals(ca, dtype="f32").cuda()
XB = workloads.signals(cb, dtype="f32").cuda()
YA, YB = torch.empty_like(XA), torch.empty_like(XB)
ZA, ZB = torch.empty_like(XA), torch.empty_like(XB)
stream = torch.cuda.current_stream()

cands = []
for R, S, W, pace, ob in itertools.product((1, 2), (2, 3, 4), (3, 4, 5, 6, 8, 10), (0, 75, 150, 250), (0, 1, 2)):
    tile = 8192 * R
    if W * (S + ob) * tile + 2048 > 227 * 1024:
        continue
    if ob == 0 and W < 6:
        continue
    cands.append((R, S, W, pace, ob))
print(json.dumps({"candidates": len(cands)}), flush=True)


def build(c):
    R, S, W, pace, ob = c
    os.environ["GFT_FMA_OBUF"] = str(ob)     # read at generation time (set_tuning) -- serialised below
    p = gft.Plan.from_config(ca, dtypes=("f32",), no_cubin_cache=True)
    try:
        p.set_tuning({kind: (R, S, W, pace)}, "f32")
    except gft.GFTError:
        return None
    return p


plans = []
for c in cands:          # generation is serial (env knob), compilation parallel
    p = build(c)
    if p is not None:
        plans.append((c, p))
os.environ.pop("GFT_FMA_OBUF", None)
t0 = time.perf_counter()
with cf.ThreadPoolExecutor(16) as ex:
    list(ex.map(lambda cp: cp[1].compile("f32", kinds=(kind,)), plans))
print(json.dumps({"compiled": len(plans), "s": round(time.perf_counter() - t0, 1)}), flush=True)

ref = pa.forward(XA) if kind == 0 else pa.inverse(XA)
ok = []
for c, p in plans:
    y = p.forward(XA) if kind == 0 else p.inverse(XA)
    if torch.equal(y, ref):
        ok.append((c, p))
    else:
        print(json.dumps({"cand": c, "error": "not bit-identical"}), flush=True)
del ref, y


def timed(p):
    f, i = (p, pa) if kind == 0 else (pa, p)

    def step():
        f.forward(XA, YA, stream)
        pb.forward(XB, YB, stream)
        i.inverse(YA, ZA, stream)
        pb.inverse(YB, ZB, stream)
    torch.cuda.synchronize()
    time.sleep(0.6)
    for _ in range(5):
        step()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20):
        step()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / 20


res = {}
allp = [("default", pa)] + ok
for _ in range(2):
    for c, p in allp:
        res[c] = min(res.get(c, 1e9), timed(p))
for c, ms in sorted(res.items(), key=lambda kv: kv[1]):
    print(json.dumps({"cand": c, "step_ms": round(ms, 5)}), flush=True)
