"""cfg5a forward vs inverse with the same FMA-skeleton geometry (R, S, W, pace, obuf) -- the
inverse reaches 1.03 of the copy peak with 2,2,3,150,2, the forward 0.84 (r02_geo_confirm.log).
Launches each kernel 3 times back to back (for ncu) and prints CUDA-event GB/s outside ncu.
python asym_probe.py R S W pace obuf"""
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
for kind, f in ((0, p.forward), (1, p.inverse)):
    for _ in range(3):
        f(X, Y)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20):
        f(X, Y)
    b.record()
    b.synchronize()
    print(p.kernel_name(kind, "f32"), round(2 * cfg.batch * 64 * 4 / (a.elapsed_time(b) / 20) / 1e6, 1), "GB/s", flush=True)
