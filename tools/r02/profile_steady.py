"""Back-to-back launches for the steady-state ncu traffic capture: each of the headline
workload's four kernels (cfg5a / cfg5b forward and inverse) launched 6 times in a row on
device-resident inputs > L2.  Under `ncu --cache-control none` the dirty L2 lines one launch
leaves behind are written back during the next, so the mean DRAM bytes of launches 2..6 is
the steady-state traffic per launch (a single cold launch under-counts writes)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_1907_07875_b200 import gft  # noqa: E402

for name in ("cfg5a", "cfg5b"):
    cfg = workloads.config(name)
    p = gft.Plan.from_config(cfg, dtypes=("f32",))
    X = torch.randn(cfg.batch, cfg.n, device="cuda")
    Y = torch.empty_like(X)
    for kind, f in ((0, p.forward), (1, p.inverse)):
        print(name, kind, p.kernel_name(kind, "f32"), flush=True)
        for _ in range(6):
            f(X, Y)
        torch.cuda.synchronize()
