"""cfg5a fwd-only then inv-only loops (6 launches each) with one geometry, for a steady-state
ncu capture (--cache-control none).  python asym_probe3.py R S W pace obuf"""
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
for f in (p.forward, p.inverse):
    for _ in range(6):
        f(X, Y)
    torch.cuda.synchronize()
