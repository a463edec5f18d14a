"""Does the relative placement of the input and output buffers matter?  One 4 GiB arena; X at
offset 0, Y at offset D for a list of D (power-of-two and odd multiples of 1 MiB / 64 KiB /
4 KiB); times cfg5b forward (tcgen05 IO-split), cfg5a forward / inverse (CUDA-core skeleton)
and a plain torch copy of the same bytes, 20 back-to-back launches, best of 3, interleaved."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_1907_07875_b200 import gft  # noqa: E402

MiB = 1 << 20
arena = torch.empty(4096 * MiB // 4, dtype=torch.float32, device="cuda")
base = arena.data_ptr()
print(json.dumps({"arena_base_mod_2MiB": base % (2 * MiB), "arena_base_mod_1GiB": base % (1 << 30)}))


def view(off_bytes, rows, n):
    o = off_bytes // 4
    return arena[o:o + rows * n].view(rows, n)


def bw(fn, nbytes):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20):
            fn()
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b) / 20)
    return round(nbytes / best / 1e6, 1)


cases = []
for name in ("cfg5b", "cfg5a"):
    cfg = workloads.config(name)
    p = gft.Plan.from_config(cfg, dtypes=("f32",))
    cases.append((name, cfg, p))
arena.normal_()
offs = [512, 768, 1024, 1280, 1536, 2048, 512 + 1, 1024 + 1, 1024 + 2, 1024 + 16, 1024 + 64, 1024 + 128, 1024 + 256,
        1024 + 0.0625, 1024 + 0.004, 2048 + 0.5, 0]
for d in offs:
    D = int(d * MiB)
    row = {"Y_minus_X_MiB": d}
    for name, cfg, p in cases:
        nb = cfg.batch * cfg.n * 4
        if D != 0 and D < nb:
            continue
        X, Y = view(0, cfg.batch, cfg.n), view(D, cfg.batch, cfg.n)
        row[name + "_fwd"] = bw(lambda: p.forward(X, Y), 2 * nb)
        row[name + "_inv"] = bw(lambda: p.inverse(X, Y), 2 * nb)
        if D != 0:
            row[name + "_copy"] = bw(lambda: Y.copy_(X), 2 * nb)
    print(json.dumps(row), flush=True)
