"""Launch generated kernels in a single process (one ncu run captures them all:
ncu --set full -k regex:gft_ -s <2*i> ... or -c <2 * number of specs>).

  python tools/profile_many.py rh0:0 rh1:0 ap7:0 ...     (spec = <plan>:<kind>)
<plan> as in tools/profile_kernel.py (cfgN, rhI, apI).  Each kernel is launched twice; the
printed CUDA-event time is the second launch (never report a number taken under ncu)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def make_plan(name, gft, workloads):
    if name.startswith("rh"):
        case = workloads.RIGHT_HAAR_BENCH_CASES[int(name[2:])]
        n, s, d, w, loops, norm = workloads.right_haar_bench_graph(case)
        return gft.Plan(n, s, d, w, loops, dtypes=(case[4],), normalized=norm), n, case[4], 1 << 20
    if name.startswith("ap"):
        label, variant, kw = workloads.approx_bench_plans()[int(name[2:])]
        s, d, w = workloads.APPROX_BENCH_GRAPHS[label][0]()
        kw = dict(kw)
        phi = kw.pop("phi")
        return gft.Plan(64, s, d, w, None, phi, dtypes=("f32",), **kw), 64, "f32", 1 << 21
    cfg = workloads.config(name)
    return gft.Plan.from_config(cfg, dtypes=(cfg.dtypes[0],)), cfg.n, cfg.dtypes[0], cfg.batch


def main():
    import torch
    import workloads
    from paper_1907_07875_b200 import gft
    out = []
    for spec in sys.argv[1:]:
        name, kind = spec.split(":")
        kind = int(kind)
        plan, n, dt, B = make_plan(name, gft, workloads)
        X = torch.randn(B, n, device="cuda", dtype=torch.float64 if dt == "f64" else torch.float32)
        Y = torch.empty_like(X)
        fn = [plan.forward, plan.inverse, plan.dense_forward, plan.dense_inverse][kind]
        fn(X, Y)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn(X, Y)
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e)
        out.append({"spec": spec, "kernel": plan.kernel_name(kind, dt), "ms": ms,
                    "gbs": 2 * B * n * X.element_size() / ms / 1e6})
        del X, Y
        plan.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
