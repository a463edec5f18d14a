"""e2e (gft_execute_host) sweep over chunk size and slot count on cfg2: forward + inverse of
2^22 signals from / to pinned host memory, CUDA-event timed on the caller stream."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import workloads
    from paper_1907_07875_b200 import gft
    cfg = workloads.config("cfg2")
    plan = gft.Plan.from_config(cfg, dtypes=("f32",))
    n, B = cfg.n, cfg.batch
    Xh = torch.randn(B, n).pin_memory()
    Yh, Zh = torch.empty_like(Xh).pin_memory(), torch.empty_like(Xh).pin_memory()
    stream = torch.cuda.current_stream().cuda_stream
    for log2c, slots in [(c, k) for c in (16, 17, 18, 19) for k in (2, 3, 4)]:
            chunk = 1 << log2c
            ws = torch.empty(slots * chunk * n, device="cuda")
            step = lambda: (plan.execute_host(0, Xh, Yh, ws, chunk, stream),
                            plan.execute_host(1, Yh, Zh, ws, chunk, stream))
            for _ in range(2):
                step()
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(4):
                step()
            e.record()
            torch.cuda.synchronize()
            ms = s.elapsed_time(e) / 4
            err = float(((Zh.double() - Xh.double()).norm(dim=1) / Xh.double().norm(dim=1)).max())
            Zh.zero_()
            print(json.dumps({"chunk": chunk, "slots": slots, "ms": round(ms, 3),
                              "each_dir_gbs": round(2 * B * n * 4 / (ms * 1e6), 1),
                              "roundtrip_err": err}), flush=True)


if __name__ == "__main__":
    main()
