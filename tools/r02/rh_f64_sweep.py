"""Right-Haar 12|20 f64 plan (n = 32): forward + inverse pair in both regimes for a list of FMA
geometries "R,S,W,pace,obuf" (or "default" / "copy"), as tools/r02/regime_sweep.py does for the
BASELINE configs."""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_1907_07875_b200 import gft  # noqa: E402

case = workloads.RIGHT_HAAR_BENCH_CASES[3]
n, s, d, w, loops, norm = workloads.right_haar_bench_graph(case)
X = torch.randn(1 << 20, n, device="cuda", dtype=torch.float64)
Y, Z = torch.empty_like(X), torch.empty_like(X)
nbytes = 4 * X.numel() * 8
stream = torch.cuda.current_stream()


def make(spec):
    if spec == "copy":
        return None
    if spec == "default":
        return gft.Plan(n, s, d, w, loops, dtypes=("f64",), normalized=norm)
    R, S, W, pace, ob = (int(v) for v in spec.split(","))
    os.environ["GFT_FMA_OBUF"] = str(ob)
    p = gft.Plan(n, s, d, w, loops, dtypes=("f64",), normalized=norm, no_cubin_cache=True)
    p.set_tuning({0: (R, S, W, pace), 1: (R, S, W, pace)}, "f64")
    os.environ.pop("GFT_FMA_OBUF")
    return p


def stepper(p):
    if p is None:
        return lambda: (Y.copy_(X), Z.copy_(Y))
    return lambda: (p.forward(X, Y, stream), p.inverse(Y, Z, stream))


def timed(step, k):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(k):
        step()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / k


made = []
for c in sys.argv[1:]:
    try:
        made.append((c, make(c)))
    except gft.GFTError as e:
        print(json.dumps({"cand": c, "skipped": str(e)[:80]}), flush=True)
res = {c: ([], []) for c, _ in made}
for _ in range(3):
    for c, p in made:
        st = stepper(p)
        torch.cuda.synchronize()
        time.sleep(1.5)
        for _ in range(5):
            st()
        torch.cuda.synchronize()
        res[c][0].append(timed(st, 20))
        t0 = time.perf_counter()
        while time.perf_counter() - t0 < 1.5:
            timed(st, 200)
        res[c][1].append(statistics.mean(timed(st, 200) for _ in range(3)))
cb, cs = (statistics.median(res["copy"][i]) for i in (0, 1))
for c, _ in made:
    b, su = statistics.median(res[c][0]), statistics.median(res[c][1])
    print(json.dumps({"cand": c, "burst_gbs": round(nbytes / b / 1e6, 1), "sustained_gbs": round(nbytes / su / 1e6, 1),
                      "burst_vs_copy": round(cb / b, 4), "sustained_vs_copy": round(cs / su, 4)}), flush=True)
