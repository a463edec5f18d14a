"""cfg5a fwd / inv back-to-back interaction: for a geometry (R S W pace obuf), time 20 launches
of fwd only, inv only, and alternating fwd/inv (per-kernel time = total / launches), plus a
run with an event between launches; GFT_PDL=0 in the environment disables programmatic
dependent launch.  python asym_probe2.py R S W pace obuf"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_1907_07875_b200 import gft  # noqa: E402

R, S, W, pace, ob = (int(v) for v in sys.argv[1:6])
os.environ["GFT_FMA_OBUF"] = str(ob)
cfg = workloads.config("cfg5a")
p = gft.Plan.from_config(cfg, dtypes=("f32",), no_cubin_cache=True)
p.set_tuning({0: (R, S, W, pace), 1: (R, S, W, pace)}, "f32")
X = torch.randn(cfg.batch, cfg.n, device="cuda")
Y = torch.empty_like(X)
Z = torch.empty_like(X)
nb = 2 * cfg.batch * 64 * 4


def run(seq, reps=10):
    for f in seq:
        f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        for f in seq:
            f()
    b.record()
    b.synchronize()
    return round(nb / (a.elapsed_time(b) / (reps * len(seq))) / 1e6, 1)


fw = lambda: p.forward(X, Y)    # noqa: E731
iv = lambda: p.inverse(X, Z)    # noqa: E731
iv2 = lambda: p.inverse(Y, Z)   # noqa: E731
print(dict(geom=sys.argv[1:6], pdl=os.environ.get("GFT_PDL", "1"), fwd_only=run([fw, fw]), inv_only=run([iv, iv]),
           alt=run([fw, iv]), chain=run([fw, iv2]), fwd_x_then_inv_x=run([fw, iv])), flush=True)
