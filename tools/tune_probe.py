"""gft_plan_tune on graphs outside the tuning table: default kernel vs pacing-only vs
geometry + pacing (GFT_TUNE_GEOMETRY), forward kernel, back-to-back GB/s on 2^21 signals.
python tools/tune_probe.py  (B200, under gpurun)"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_1907_07875_b200 import gft  # noqa: E402


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


def mirror_graph(n, p, seed):
    rng = np.random.default_rng(seed)
    s_, d_, w_ = [], [], []
    h = n // 2
    for i in range(h):
        for j in range(i + 1, h):
            if rng.random() < p:
                w = rng.uniform(0.5, 2.0)
                s_ += [i, n - 1 - i]
                d_ += [j, n - 1 - j]
                w_ += [w, w]
        s_.append(i)
        d_.append(n - 1 - i)
        w_.append(rng.uniform(0.5, 2.0))
    return np.array(s_, np.int32), np.array(d_, np.int32), np.array(w_)


cases = []
for n, p, seed in ((12, 0.4, 1), (24, 0.3, 2), (40, 0.2, 3), (48, 0.15, 4), (72, 0.1, 5)):
    cases.append(("mirror n=%d" % n, n, mirror_graph(n, p, seed)))
for n in (20, 36):                                  # cycles (Lemma 1 pairing, deep recursion)
    src = np.arange(n, dtype=np.int32)
    cases.append(("cycle n=%d" % n, n, (src, (src + 1) % n, np.ones(n))))
for name, n, (s_, d_, w_) in cases:
    X = torch.randn(1 << 21, n, device="cuda")
    Y = torch.empty_like(X)
    nb = 2 * X.numel() * 4
    row = {"graph": name}
    for tag, geo in (("default", None), ("pace", False), ("geometry+pace", True)):
        plan = gft.Plan(n, s_, d_, w_, dtypes=("f32",))
        t = time.perf_counter()
        ch = None if geo is None else plan.tune("f32", (0,), X, Y, geometry=geo)
        row[tag] = {"gbs": round(nb / b2b(lambda: plan.forward(X, Y)) / 1e6, 1),
                    "choice": None if ch is None else ch.get(0), "tune_s": round(time.perf_counter() - t, 2),
                    "kernel": plan.kernel_name(0, "f32")[:30]}
        plan.close()
    print(json.dumps(row), flush=True)
