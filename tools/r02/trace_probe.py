"""Phase trace of a tcgen05 GFT kernel (variant knobs in the environment): optionally heats the
GPU first with the untraced kernel back to back for `heat` seconds (power-capped clock), then
launches the traced build (GFT_TC_TRACE=1) a few times; the kernel printf's per-tile clock64
stamps of CTAs 0 and 1 (see kernel_tc3_skeleton.cuh).
  python trace_probe.py <cfg> <launches> [heat_seconds]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import workloads  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import probe_plans  # noqa: E402
from paper_1907_07875_b200 import gft  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg5b"
n_launch = int(sys.argv[2]) if len(sys.argv) > 2 else 4
heat = float(sys.argv[3]) if len(sys.argv) > 3 else 0.0
os.environ.pop("GFT_TC_TRACE", None)
p0, n, batch, _ = probe_plans.make(name, no_cubin_cache=True)
os.environ["GFT_TC_TRACE"] = "1"
p, _, _, _ = probe_plans.make(name, no_cubin_cache=True)
X = torch.randn(batch, n, device="cuda")
Y = torch.empty_like(X)
p.compile("f32", kinds=(0,))
p0.forward(X, Y)
torch.cuda.synchronize()
if heat > 0:
    t = time.perf_counter()
    while time.perf_counter() - t < heat:
        for _ in range(200):
            p0.forward(X, Y)
        torch.cuda.synchronize()
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
    print("sm_mhz_before_trace", pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM), flush=True)
print("kernel", p.kernel_name(0, "f32"), flush=True)
for _ in range(n_launch):
    p.forward(X, Y)
torch.cuda.synchronize()
