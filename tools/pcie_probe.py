"""PCIe roof on the GPU box: pinned H2D, D2H and both directions concurrently (torch
copies on two streams), and gft_execute_host at several chunk sizes (cfg2 forward).

  python tools/pcie_probe.py  ->  one JSON line
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import workloads  # noqa: E402
from paper_1907_07875_b200 import gft as G  # noqa: E402


def timed(fn, iters=5):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def main():
    nbytes = 256 << 20
    h_src = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    h_dst = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d_a = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    d_b = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    out = {}
    out["h2d_gbs"] = nbytes / timed(lambda: d_a.copy_(h_src, non_blocking=True)) / 1e6
    out["d2h_gbs"] = nbytes / timed(lambda: h_dst.copy_(d_b, non_blocking=True)) / 1e6

    def both():
        cur = torch.cuda.current_stream()
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            d_a.copy_(h_src, non_blocking=True)
        with torch.cuda.stream(s2):
            h_dst.copy_(d_b, non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)
    out["bidir_each_gbs"] = nbytes / timed(both) / 1e6
    cfg = workloads.config("cfg2")
    plan = G.Plan.from_config(cfg, dtypes=("f32",))
    X = workloads.signals(cfg, dtype="f32").pin_memory()
    Y = torch.empty_like(X).pin_memory()
    stream = torch.cuda.current_stream().cuda_stream
    rows = {}
    for slots in (2, 3, 4):
        for lg in (16, 17, 18, 19):
            chunk = 1 << lg
            ws = torch.empty(slots * chunk * cfg.n, dtype=torch.float32, device="cuda")
            ms = timed(lambda: plan.execute_host(0, X, Y, ws, chunk, stream))
            rows["%d slots x %d rows" % (slots, chunk)] = {"ms": round(ms, 3),
                                                           "each_dir_gbs": round(X.numel() * 4 / ms / 1e6, 1)}
    out["execute_host_cfg2_fwd"] = rows
    print(json.dumps(out))


if __name__ == "__main__":
    main()
