"""The tcgen05 dense comparison kernels (dense_tc plans) of cfg5a / cfg5b: kernel names and
back-to-back GB/s of the dense forward and inverse; GFT_TC_IOSPLIT=0 in the environment gives
the plain CTA-pair kernel for comparison."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_1907_07875_b200 import gft  # noqa: E402

for name in ("cfg5a", "cfg5b"):
    cfg = workloads.config(name)
    p = gft.Plan.from_config(cfg, dtypes=("f32",), dense_tc=True, no_cubin_cache=True)
    X = torch.randn(cfg.batch, cfg.n, device="cuda")
    Y = torch.empty_like(X)
    for kind, f in ((2, p.dense_forward), (3, p.dense_inverse)):
        for _ in range(3):
            f(X, Y)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20):
            f(X, Y)
        b.record()
        b.synchronize()
        ms = a.elapsed_time(b) / 20
        print(name, p.kernel_name(kind, "f32"), round(ms, 5), "ms", round(2 * cfg.batch * cfg.n * 4 / ms / 1e6, 1), "GB/s",
              flush=True)
