"""cfg5b forward through the IO-split warp-specialised kernel and the plain pair kernel in ONE
process (one ncu run captures both): each launched twice.  Prints CUDA-event times."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import workloads  # noqa: E402
from paper_1907_07875_b200 import gft as G  # noqa: E402

cfg = workloads.config("cfg5b")
os.environ["GFT_TC_IOSPLIT"] = "1"
plans = [G.Plan.from_config(cfg, dtypes=("f32",))]
os.environ.pop("GFT_TC_IOSPLIT", None)
plans.append(G.Plan.from_config(cfg, dtypes=("f32",)))
X = torch.randn(cfg.batch, cfg.n, device="cuda")
Y = torch.empty_like(X)
out = []
for p in plans:
    p.forward(X, Y)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    p.forward(X, Y)
    e.record()
    torch.cuda.synchronize()
    out.append({"kernel": p.kernel_name(0, "f32"), "ms": s.elapsed_time(e)})
print(json.dumps(out))
