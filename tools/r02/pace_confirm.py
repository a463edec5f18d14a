"""Load-pacing confirmation for a tcgen05 warp-specialised plan: one plan per GFT_TC_LOAD_PACE_NS
value (compile-time), forward and inverse timed in interleaved rounds (best of 3 x 40 launches
per round, 3 rounds), median GB/s per pace.  python pace_confirm.py <plan> <pace> ..."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch  # noqa: E402

import probe_plans  # noqa: E402

name = sys.argv[1]
paces = [int(v) for v in sys.argv[2:]]
plans = []
for pc in paces:
    os.environ["GFT_TC_LOAD_PACE_NS"] = str(pc)
    p, n, batch, _ = probe_plans.make(name, no_cubin_cache=True)
    plans.append(p)
os.environ.pop("GFT_TC_LOAD_PACE_NS")
X = torch.randn(batch, n, device="cuda")
Y = torch.empty_like(X)
nb = 2 * batch * n * 4


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


res = {(pc, k): [] for pc in paces for k in ("fwd", "inv")}
for _ in range(3):
    for pc, p in zip(paces, plans):
        res[(pc, "fwd")].append(timed(lambda: p.forward(X, Y)))
        res[(pc, "inv")].append(timed(lambda: p.inverse(X, Y)))
print(json.dumps({"plan": name, "median_gbs": {"%d_%s" % k: round(statistics.median(v), 1) for k, v in res.items()}}))
