"""Run-to-run variation of the bench's e2e arm (gft_execute_host, cfg5 mixed, pinned host
buffers): 6 rounds of 3 steps, each timed with CUDA events, plus the PCIe roof before / after."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import workloads  # noqa: E402
from paper_1907_07875_b200 import gft  # noqa: E402

dev = torch.device("cuda", 0)
cfgs = [workloads.config("cfg5a"), workloads.config("cfg5b")]
plans = [gft.Plan.from_config(c, dtypes=("f32",)) for c in cfgs]
Xh = [workloads.signals(c, dtype="f32").pin_memory() for c in cfgs]
Yh = [torch.empty_like(x).pin_memory() for x in Xh]
Zh = [torch.empty_like(x).pin_memory() for x in Xh]
chunk = int(os.environ.get("E2E_CHUNK", 1 << 17))
slots = int(os.environ.get("E2E_SLOTS", 4))
# E2E_CHUNK_BYTES: chunks of equal BYTES for both graphs (rows = bytes / row bytes) instead of equal rows
cbytes = int(os.environ.get("E2E_CHUNK_BYTES", 0))
chunks = [cbytes // (c.n * 4) if cbytes else chunk for c in cfgs]
order = [int(v) for v in os.environ.get("E2E_ORDER", "01")]   # graph order inside each direction
wsb = [torch.empty(slots * ch * c.n, dtype=torch.float32, device=dev) for c, ch in zip(cfgs, chunks)]
stream = torch.cuda.current_stream()
gs = [torch.cuda.Stream(dev), torch.cuda.Stream(dev)]
step_bytes = sum(2 * c.batch * c.n * 4 for c in cfgs)


def e2e_step():
    for s in gs:
        s.wait_stream(stream)
    for d in (0, 1):
        for i in order:
            plans[i].execute_host(d, Xh[i] if d == 0 else Yh[i], Yh[i] if d == 0 else Zh[i], wsb[i], chunks[i], gs[i])
    for s in gs:
        stream.wait_stream(s)


print(json.dumps({"pcie_roof_before": bench.pcie_roof(dev)}), flush=True)
e2e_step()
torch.cuda.synchronize()
for r in range(6):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(3):
        e2e_step()
    b.record(stream)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 3
    print(json.dumps({"round": r, "chunks": chunks, "order": order, "slots": slots, "ms": round(ms, 3),
                      "each_dir_gbs": round(step_bytes / (ms * 1e6), 1)}), flush=True)
print(json.dumps({"pcie_roof_after": bench.pcie_roof(dev)}), flush=True)
