"""Launch one generated kernel a few times on a config's full batch (for ncu / timing).

  python tools/profile_kernel.py --config cfg2 --kind 0 --dtype f32 --iters 5
kind: 0 fast fwd, 1 fast inv, 2 dense fwd, 3 dense inv.  Prints per-launch CUDA-event
times (never report a number taken under ncu).
--config also accepts rhI (workloads.RIGHT_HAAR_BENCH_CASES[I], right Haar plan) and apI
(workloads.approx_bench_plans()[I], the Sec. VI-B plans), with 2^20 signals by default."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--kind", type=int, default=0)
    ap.add_argument("--dtype", default=None)
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--batch", type=int, default=None)
    a = ap.parse_args()
    import torch
    import workloads
    from paper_1907_07875_b200 import gft
    if a.config.startswith("rh"):
        case = workloads.RIGHT_HAAR_BENCH_CASES[int(a.config[2:])]
        n, s_, d_, w_, loops, norm = workloads.right_haar_bench_graph(case)
        dt = a.dtype or case[4]
        plan = gft.Plan(n, s_, d_, w_, loops, dtypes=(dt,), normalized=norm)
        B = a.batch or (1 << 20)
    elif a.config.startswith("ap"):
        label, variant, kw = workloads.approx_bench_plans()[int(a.config[2:])]
        s_, d_, w_ = workloads.APPROX_BENCH_GRAPHS[label][0]()
        kw = dict(kw)
        phi = kw.pop("phi")
        n, dt = 64, a.dtype or "f32"
        plan = gft.Plan(64, s_, d_, w_, None, phi, dtypes=(dt,), **kw)
        B = a.batch or (1 << 21)
    else:
        cfg = workloads.config(a.config)
        n, dt = cfg.n, a.dtype or cfg.dtypes[0]
        plan = gft.Plan.from_config(cfg, dtypes=(dt,))
        B = a.batch or cfg.batch
    X = torch.randn(B, n, device="cuda", dtype=torch.float64 if dt == "f64" else torch.float32)
    Y = torch.empty_like(X)
    fn = [plan.forward, plan.inverse, plan.dense_forward, plan.dense_inverse][a.kind]
    times = []
    for _ in range(a.iters):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn(X, Y)
        e.record()
        torch.cuda.synchronize()
        times.append(s.elapsed_time(e))
    nbytes = 2 * B * n * X.element_size()
    # back-to-back launches between two events (no idle gaps between kernels)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20):
        fn(X, Y)
    e.record()
    torch.cuda.synchronize()
    b2b = s.elapsed_time(e) / 20
    print(json.dumps({"config": a.config, "kind": a.kind, "dtype": dt, "kernel": plan.kernel_name(a.kind, dt),
                      "launch": plan.launch_config(a.kind, dt, B), "ms": times,
                      "gbs_best": nbytes / min(times) / 1e6, "b2b_ms": b2b, "b2b_gbs": nbytes / b2b / 1e6}))


if __name__ == "__main__":
    main()
