"""Host-side cost of one launch (cfg1, 4096 x 8 f32, launch-bound): wall time per call of
Plan.forward (Python binding), of the raw ctypes gft_forward with pre-marshalled arguments,
and GPU time per launch back to back and from a CUDA graph.  python tools/host_overhead_probe.py"""
import ctypes
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_1907_07875_b200 import gft  # noqa: E402

cfg = workloads.config("cfg1")
plan = gft.Plan.from_config(cfg, dtypes=("f32",))
X = torch.randn(cfg.batch, cfg.n, device="cuda")
Y = torch.empty_like(X)
N = 5000
out = {}
for _ in range(200):
    plan.forward(X, Y)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(N):
    plan.forward(X, Y)
t_py = (time.perf_counter() - t) / N
torch.cuda.synchronize()
out["python_binding_us_per_call"] = round(t_py * 1e6, 2)
lib = gft.lib()
h, px, py_ = plan._h, ctypes.c_void_p(X.data_ptr()), ctypes.c_void_p(Y.data_ptr())
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
f = lib.gft_forward
t = time.perf_counter()
for _ in range(N):
    f(h, px, py_, cfg.batch, 0, st)
t_c = (time.perf_counter() - t) / N
torch.cuda.synchronize()
out["raw_ctypes_us_per_call"] = round(t_c * 1e6, 2)
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(N):
    f(h, px, py_, cfg.batch, 0, st)
e.record()
torch.cuda.synchronize()
out["gpu_us_per_launch_b2b_raw"] = round(s.elapsed_time(e) * 1e3 / N, 2)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    for _ in range(20):
        plan.forward(X, Y)
g.replay()
torch.cuda.synchronize()
s.record()
for _ in range(50):
    g.replay()
e.record()
torch.cuda.synchronize()
out["gpu_us_per_launch_graph"] = round(s.elapsed_time(e) * 1e3 / (50 * 20), 2)
print(json.dumps(out))
