"""Headline step (5a fwd, 5b fwd, 5a inv, 5b inv) with plans generated under two or more
environments (each arg: ENV=VALUE,... or "default"), timed in interleaved rounds inside one
process (best of 3 x 20 steps per round, 7 rounds); prints median and min step time per variant."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_1907_07875_b200 import gft  # noqa: E402

ca, cb = workloads.config("cfg5a"), workloads.config("cfg5b")
XA = workloads.signals(ca, dtype="f32").cuda()
XB = workloads.signals(cb, dtype="f32").cuda()
YA, ZA, YB, ZB = (torch.empty_like(t) for t in (XA, XA, XB, XB))
variants = sys.argv[1:] or ["default"]
made = []
for v in variants:
    env = {} if v == "default" else dict(kv.split("=", 1) for kv in v.split(","))
    os.environ.update(env)
    pa = gft.Plan.from_config(ca, dtypes=("f32",), no_cubin_cache=True)
    pb = gft.Plan.from_config(cb, dtypes=("f32",), no_cubin_cache=True)
    for k in env:
        os.environ.pop(k)
    made.append((v, pa, pb))


def timed(pa, pb):
    def step():
        pa.forward(XA, YA)
        pb.forward(XB, YB)
        pa.inverse(YA, ZA)
        pb.inverse(YB, ZB)
    for _ in range(3):
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


res = {v: [] for v in variants}
for _ in range(7):
    for v, pa, pb in made:
        res[v].append(timed(pa, pb))
for v, pa, pb in made:
    print(json.dumps({"variant": v, "median_ms": round(statistics.median(res[v]), 5), "min_ms": round(min(res[v]), 5),
                      "kernels": [pb.kernel_name(0, "f32"), pb.kernel_name(1, "f32")]}), flush=True)
