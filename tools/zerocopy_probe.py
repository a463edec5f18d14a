"""Zero-copy probe: launch the generated kernels directly on pinned (UVA-mapped) HOST buffers,
so TMA / bulk copies read and write host memory over PCIe -- no staging copies, one launch
per transform, both PCIe directions busy at once.  Checks the result against the device
path and times forward + inverse host->host."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import workloads
    from paper_1907_07875_b200 import gft as G
    for name in sys.argv[1:] or ["cfg2"]:
        cfg = workloads.config(name)
        plan = G.Plan.from_config(cfg, dtypes=("f32",))
        n, B = cfg.n, cfg.batch
        Xh = torch.randn(B, n).pin_memory()
        Yh, Zh = torch.empty_like(Xh).pin_memory(), torch.empty_like(Xh).pin_memory()
        Yd = plan.forward(Xh.cuda())
        torch.cuda.synchronize()
        G.gft_forward(plan._h, Xh.data_ptr(), Yh.data_ptr(), B)
        torch.cuda.synchronize()
        same = bool(torch.equal(Yh, Yd.cpu()))
        def step():
            G.gft_forward(plan._h, Xh.data_ptr(), Yh.data_ptr(), B)
            G.gft_inverse(plan._h, Yh.data_ptr(), Zh.data_ptr(), B)
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
        print(json.dumps({"config": name, "kernel": plan.kernel_name(0, "f32"), "bit_identical_to_device": same,
                          "fwd_inv_ms": round(ms, 3), "each_dir_gbs": round(2 * B * n * 4 / (ms * 1e6), 1),
                          "roundtrip_err": err}), flush=True)


if __name__ == "__main__":
    main()
