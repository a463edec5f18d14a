"""Pinned-host copy bandwidth with 1 / 2 / 4 concurrent streams per direction: H2D only, D2H
only and both directions at once (256 MiB per direction per round, split evenly over the
streams); CUDA events on the default stream.  Is one copy stream per direction the roof?"""
import json
import torch

NB = 256 << 20
hs = torch.empty(NB, dtype=torch.uint8).pin_memory()
hd = torch.empty(NB, dtype=torch.uint8).pin_memory()
da = torch.empty(NB, dtype=torch.uint8, device="cuda")
db = torch.empty(NB, dtype=torch.uint8, device="cuda")


def run(k, h2d, d2h, reps=4):
    ss = [torch.cuda.Stream() for _ in range(2 * k)]
    part = NB // k
    cur = torch.cuda.current_stream()

    def once():
        for s in ss:
            s.wait_stream(cur)
        for i in range(k):
            if h2d:
                with torch.cuda.stream(ss[i]):
                    da[i * part:(i + 1) * part].copy_(hs[i * part:(i + 1) * part], non_blocking=True)
            if d2h:
                with torch.cuda.stream(ss[k + i]):
                    hd[i * part:(i + 1) * part].copy_(db[i * part:(i + 1) * part], non_blocking=True)
        for s in ss:
            cur.wait_stream(s)
    once()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        once()
    b.record()
    torch.cuda.synchronize()
    return round(NB / (a.elapsed_time(b) / reps) / 1e6, 1)


for k in (1, 2, 4):
    print(json.dumps({"streams_per_dir": k, "h2d_gbs": run(k, True, False), "d2h_gbs": run(k, False, True),
                      "bidir_each_gbs": run(k, True, True)}), flush=True)
