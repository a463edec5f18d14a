#!/usr/bin/env python
"""Benchmark of the fused fast-GFT hot path on B200 (contract: see DESIGN.md §Measurement).

  python bench.py [--gpus N --steps K --warmup W] [--config cfg2] [--impl ours|reference]

One step = one fast forward GFT + one fast inverse GFT over the config's whole batch
(rows H1-H6 of SURVEY §8(a)); the dense U^T x kernel (H7) is timed beside it.
Default workload = BASELINE.json configs[1] (cfg2: symmetric line N=16, 2^22 signals).
Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "fast-GFT signals/sec and achieved HBM GB/s (% roofline) vs dense Uᵀx"
KIND_NAMES = {0: "fast_fwd", 1: "fast_inv", 2: "dense_fwd", 3: "dense_inv"}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (copy kernel, measured)"
    except Exception:
        return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


def load_traffic(kernel_prefix, config, dtype="f32", kernel_name=None):
    """dram bytes per launch from the committed ncu --set full summary, if any (only when
    the captured kernel is the one being timed: same generated-kernel name)."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as f:
            d = json.load(f)
        for row in d.get("kernels", []):
            if (row.get("config") == config and row.get("kind") == kernel_prefix
                    and row.get("tag") in (None, dtype)
                    and (kernel_name is None or row.get("kernel") == kernel_name)):
                return row.get("dram_bytes_per_launch")
    except Exception:
        pass
    return None


class ClockSampler:
    """NVML sampling of SM clocks / throttle reasons while the GPU works."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, device_index):
        self.samples = []
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover
            self.err = str(e)

    def _run(self):
        while not self._stop.is_set():
            try:
                t = time.perf_counter()
                sm = self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM)
                fn = getattr(self.nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                    self.nv.nvmlDeviceGetCurrentClocksThrottleReasons
                rs = fn(self.h)
                self.samples.append((t, sm, rs))
            except Exception:
                pass
            time.sleep(0.002)

    def start(self):
        if self.ok:
            self.th = threading.Thread(target=self._run, daemon=True)
            self.th.start()

    def stop(self):
        if self.ok:
            self._stop.set()
            self.th.join()

    def summary(self, t0, t1):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "note": "nvml unavailable"}
        win = [s for s in self.samples if t0 <= s[0] <= t1]
        note = "samples inside timed region"
        if not win:   # timed region shorter than the sampling period: nearest samples
            win = sorted(self.samples, key=lambda s: min(abs(s[0] - t0), abs(s[0] - t1)))[:5]
            note = "timed region shorter than sampling period; nearest samples"
        reasons = set()
        for _, _, r in win:
            for bit, name in self.REASONS.items():
                if r & bit and name != "gpu_idle":
                    reasons.add(name)
        return {"sm_mhz": statistics.median([s[1] for s in win]) if win else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(reasons), "samples": len(win),
                "note": note}


from paper_1907_07875_b200.dist import barrier, dist_env, max_over_ranks  # noqa: E402


def fma_peak_per_s(dtype, sm_mhz=1965.0, sms=148):
    """Lane-FMA issue peak: FFMA with an immediate operand (the form the generated kernels use)
    issues 1 warp instruction / clk / SMSP (B300_MICROARCH.md "FFMA imm-form rt_SMSP=1"), i.e.
    128 lane-FMAs / clk / SM; DFMA runs at half that on B200.  sm_mhz = the max SM clock."""
    return sms * (128 if dtype == "f32" else 64) * sm_mhz * 1e6


def time_kernel(fn, stream, warmup, iters):
    import torch
    for _ in range(warmup):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record(stream)
    for _ in range(iters):
        fn()
    e.record(stream)
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def time_graph(fn, iters):
    """Per-launch device time of `fn` replayed from a captured CUDA graph (removes the host
    launch overhead that dominates tiny workloads such as cfg1)."""
    import torch
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(iters):
            fn()
    g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    g.replay()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def config_table(args, stream, hbm, device):
    """Every BASELINE config: fast fwd/inv and dense fwd/inv, device-resident N(0,1)."""
    import torch
    import workloads
    from paper_1907_07875_b200 import gft
    rows = []
    for name, dtype in (("cfg1", "f32"), ("cfg1@2^24", "f32"), ("cfg2", "f32"), ("cfg2b", "f32"),
                        ("cfg3", "f32"), ("cfg4", "f32"), ("cfg4", "f64"), ("cfg5a", "f32"), ("cfg5b", "f32")):
        # cfg1@2^24: SURVEY §8(d)'s optional extra -- the N = 8 line graph at 2^24 signals, a
        # bandwidth point for the smallest graph (cfg1 itself is launch-bound)
        cfg = workloads.config(name.split("@")[0])
        if "@" in name:
            cfg.batch = 1 << 24
        plan = gft.Plan.from_config(cfg, dtypes=(dtype,))
        tdt = torch.float64 if dtype == "f64" else torch.float32
        g = torch.Generator(device=device).manual_seed(cfg.seed)
        X = torch.randn(cfg.batch, cfg.n, generator=g, device=device, dtype=tdt)
        Y = torch.empty_like(X)
        esz = X.element_size()
        nbytes = 2 * cfg.batch * cfg.n * esz
        row = {"config": name, "dtype": dtype, "n": cfg.n, "batch": cfg.batch,
               "units_per_level": plan.info()["units_per_level"], "leaves": plan.leaf_sizes()}
        for kind, f in ((0, plan.forward), (1, plan.inverse), (2, plan.dense_forward),
                        (3, plan.dense_inverse)):
            ms = time_kernel(lambda: f(X, Y, stream), stream, 3, args.table_iters)
            row[KIND_NAMES[kind]] = {"ms": round(ms, 5), "gbs": round(nbytes / ms / 1e6, 1),
                                     "frac": round(nbytes / ms / 1e6 / hbm, 4),
                                     "signals_per_s": cfg.batch / ms * 1e3}
        if cfg.batch * cfg.n * esz <= (64 << 20):   # small workloads: launch-bound, replay a graph
            row["fast_fwd"]["graph_ms"] = round(time_graph(lambda: plan.forward(X, Y), 50), 5)
            # the forward -> inverse pair, also from a graph
            Z1 = torch.empty_like(X)
            row["fwd_inv_pair_graph_ms"] = round(time_graph(lambda: (plan.forward(X, Y), plan.inverse(Y, Z1)), 50), 5)
        # the dense kernel is FMA-issue-bound for n >= 64: its fraction of the lane-FMA peak
        row["dense_fwd"]["fma_frac"] = round(cfg.n * cfg.n * cfg.batch / (row["dense_fwd"]["ms"] * 1e-3)
                                             / fma_peak_per_s(dtype), 4)
        row["fast_vs_dense_fwd"] = round(row["dense_fwd"]["ms"] / row["fast_fwd"]["ms"], 3)
        row["fast_vs_dense_inv"] = round(row["dense_inv"]["ms"] / row["fast_inv"]["ms"], 3)
        # fused graph filter U diag(exp(-lambda)) U^T (one pass) vs forward + inverse (two)
        filt = gft.Filter(plan, np.exp(-plan.eigenvalues()), dtypes=(dtype,))
        ms = time_kernel(lambda: filt.apply(X, Y, stream), stream, 3, args.table_iters)
        row["filter"] = {"ms": round(ms, 5), "gbs": round(nbytes / ms / 1e6, 1),
                         "frac": round(nbytes / ms / 1e6 / hbm, 4), "signals_per_s": cfg.batch / ms * 1e3,
                         "kernel": filt.kernel_name(dtype)}
        row["fused_filter_vs_two_pass"] = round((row["fast_fwd"]["ms"] + row["fast_inv"]["ms"]) / ms, 3)
        if not args.no_tune and cfg.batch * cfg.n * esz > (64 << 20):
            # measured geometry + pacing (gft_filter_tune), then re-timed
            ch = filt.tune(X, Y, dtype, stream=stream, geometry=True)
            if ch is not None:
                ms = time_kernel(lambda: filt.apply(X, Y, stream), stream, 3, args.table_iters)
                row["filter_tuned"] = {"ms": round(ms, 5), "gbs": round(nbytes / ms / 1e6, 1),
                                       "frac": round(nbytes / ms / 1e6 / hbm, 4), "geometry_pace": ch}
        # cuBLAS SGEMM/DGEMM with TF32 disabled (SURVEY §7 step 6 cross-check of "dense")
        U = torch.from_numpy(plan.basis()).to(device=device, dtype=tdt)
        tf32 = torch.backends.cuda.matmul.allow_tf32
        torch.backends.cuda.matmul.allow_tf32 = False
        ms = time_kernel(lambda: torch.matmul(X, U, out=Y), stream, 3, args.table_iters)
        torch.backends.cuda.matmul.allow_tf32 = tf32
        row["cublas_fwd"] = {"ms": round(ms, 5), "gbs": round(nbytes / ms / 1e6, 1),
                             "frac": round(nbytes / ms / 1e6 / hbm, 4)}
        row["fast_vs_best_dense_fwd"] = round(min(row["dense_fwd"]["ms"], ms) / row["fast_fwd"]["ms"], 3)
        if dtype == "f32" and cfg.n % 32 == 0:
            # dense U^T x as one tcgen05 3xTF32 leaf: the strongest dense kernel (HBM-bound too)
            dplan = gft.Plan.from_config(cfg, dtypes=(dtype,), dense_tc=True)
            ms = time_kernel(lambda: dplan.dense_forward(X, Y, stream), stream, 3, args.table_iters)
            row["dense_tc_fwd"] = {"ms": round(ms, 5), "gbs": round(nbytes / ms / 1e6, 1),
                                   "frac": round(nbytes / ms / 1e6 / hbm, 4),
                                   "kernel": dplan.kernel_name(2, dtype)}
            row["fast_vs_dense_tc_fwd"] = round(ms / row["fast_fwd"]["ms"], 3)
            dplan.close()
        if not args.no_tune and cfg.batch * cfg.n * esz > (64 << 20):
            # measured geometry + pacing of the fast kernels (gft_plan_tune), then re-timed:
            # shows whether the committed tuning table still holds on this box
            ch = plan.tune(dtype, (0, 1), X, Y, stream=stream, geometry=True)
            for kind, f in ((0, plan.forward), (1, plan.inverse)):
                if kind in ch:
                    ms = time_kernel(lambda: f(X, Y, stream), stream, 3, args.table_iters)
                    row[KIND_NAMES[kind] + "_tuned"] = {"ms": round(ms, 5), "gbs": round(nbytes / ms / 1e6, 1),
                                                        "frac": round(nbytes / ms / 1e6 / hbm, 4),
                                                        "geometry_pace": ch[kind]}
        rows.append(row)
        del X, Y
        filt.close()
        plan.close()
    return rows


def mixed_cfg5_row(args, stream, hbm, device):
    """configs[4] as one mixed batch: the cycle C64 (cfg5a) and the bipartite 128-node graph
    (cfg5b), 2^20 signals each, forward of both per step -- back to back on one stream
    (programmatic dependent launch overlaps the tails) and concurrently on two streams --
    with the dense kernels of both timed alongside."""
    import torch
    import workloads
    from paper_1907_07875_b200 import gft
    ca, cb = workloads.config("cfg5a"), workloads.config("cfg5b")
    pa, pb = gft.Plan.from_config(ca, dtypes=("f32",)), gft.Plan.from_config(cb, dtypes=("f32",))
    g = torch.Generator(device=device).manual_seed(ca.seed)
    Xa = torch.randn(ca.batch, ca.n, generator=g, device=device)
    Xb = torch.randn(cb.batch, cb.n, generator=g, device=device)
    Ya, Yb = torch.empty_like(Xa), torch.empty_like(Xb)
    nbytes = 2 * 4 * (ca.batch * ca.n + cb.batch * cb.n)
    sig = ca.batch + cb.batch
    row = {"config": "cfg5 mixed (cfg5a + cfg5b)", "batch": sig}

    def rec(ms):
        return {"ms": round(ms, 5), "gbs": round(nbytes / ms / 1e6, 1), "frac": round(nbytes / ms / 1e6 / hbm, 4),
                "signals_per_s": sig / ms * 1e3}

    row["fast_fwd_one_stream"] = rec(time_kernel(lambda: (pa.forward(Xa, Ya, stream), pb.forward(Xb, Yb, stream)),
                                                 stream, 3, args.table_iters))
    s2 = torch.cuda.Stream(device)

    def two_streams():
        s2.wait_stream(stream)
        pa.forward(Xa, Ya, stream)
        with torch.cuda.stream(s2):
            pb.forward(Xb, Yb, s2)
        stream.wait_stream(s2)

    row["fast_fwd_two_streams"] = rec(time_kernel(two_streams, stream, 3, args.table_iters))
    row["dense_fwd_one_stream"] = rec(time_kernel(lambda: (pa.dense_forward(Xa, Ya, stream),
                                                           pb.dense_forward(Xb, Yb, stream)),
                                                  stream, 3, args.table_iters))
    row["fast_vs_dense"] = round(row["dense_fwd_one_stream"]["ms"] / row["fast_fwd_one_stream"]["ms"], 3)
    pa.close()
    pb.close()
    return row


def right_haar_table(args, stream, hbm, device):
    """Right Haar stages: plans with / without them on bipartite graphs
    whose Laplacian diagonal is constant, device-resident N(0,1), 2^20 signals."""
    import torch
    import workloads
    from paper_1907_07875_b200 import gft
    rows = []
    for case in workloads.RIGHT_HAAR_BENCH_CASES:
        label, dtype = case[0], case[4]
        n, s, d, w, loops, norm = workloads.right_haar_bench_graph(case)
        tdt = torch.float64 if dtype == "f64" else torch.float32
        batch = 1 << 20
        X = torch.randn(batch, n, generator=torch.Generator(device=device).manual_seed(5), device=device,
                        dtype=tdt)
        Y = torch.empty_like(X)
        nbytes = 2 * batch * n * X.element_size()
        row = {"graph": label, "dtype": dtype, "n": n, "batch": batch}
        for tag, rh in (("right_haar", True), ("one_block", False)):
            plan = gft.Plan(n, s, d, w, loops, dtypes=(dtype,), normalized=norm, right_haar=rh)
            info = plan.info()
            r = {"leaves": plan.leaf_sizes(), "pairs": info["n_right_pairs"], "mults": info["mults"],
                 "adds": info["adds"], "kernel": plan.kernel_name(0, dtype)}
            for k, f in ((0, plan.forward), (1, plan.inverse)):
                ms = time_kernel(lambda: f(X, Y, stream), stream, 3, args.table_iters)
                r[KIND_NAMES[k]] = {"ms": round(ms, 5), "gbs": round(nbytes / ms / 1e6, 1),
                                    "frac": round(nbytes / ms / 1e6 / hbm, 4)}
            # measured pacing (gft_plan_tune) for FMA-skeleton kernels, then re-timed
            paces = plan.tune(dtype, (0, 1), X, Y, stream=stream)
            for k, f in ((0, plan.forward), (1, plan.inverse)):
                if k in paces:
                    ms = time_kernel(lambda: f(X, Y, stream), stream, 3, args.table_iters)
                    r[KIND_NAMES[k] + "_tuned"] = {"ms": round(ms, 5), "gbs": round(nbytes / ms / 1e6, 1),
                                                   "frac": round(nbytes / ms / 1e6 / hbm, 4),
                                                   "geometry_pace": paces[k]}
            row[tag] = r
            plan.close()
        row["right_vs_one_block_fwd"] = round(row["one_block"]["fast_fwd"]["ms"] / row["right_haar"]["fast_fwd"]["ms"], 3)
        rows.append(row)
        del X, Y
    return rows


def approx_table(args, stream, hbm, device):
    """Sec. VI-B comparison on B200: matrix GFT, Haar + matrix (exact fast
    GFT), approximate GFT (J Givens layers) and Haar + approximate, each with its kernel time
    and the paper's error metrics delta / epsilon against the exact plan basis (M = 20000
    U[0,1] signals).  fp32, 2^21 device-resident signals (> L2)."""
    import torch
    import workloads
    from paper_1907_07875_b200 import gft
    batch = 1 << 21
    Xs = np.random.default_rng(0).uniform(0.0, 1.0, (20000, 64))
    X = torch.rand(batch, 64, generator=torch.Generator(device=device).manual_seed(6), device=device)
    Y = torch.empty_like(X)
    nbytes = 2 * batch * 64 * 4
    rows, exact = [], {}

    def delta(Uh, U):
        return float(np.linalg.norm(np.abs(Uh.T @ U) - np.eye(64)) / 8.0)

    def eps(Uh, U):
        dd = np.abs(Xs @ U) - np.abs(Xs @ Uh)
        return float(np.sum(dd * dd) / Xs.shape[0])

    for label, variant, kw in workloads.approx_bench_plans():
        s, d, w = workloads.APPROX_BENCH_GRAPHS[label][0]()
        kw = dict(kw)
        phi = kw.pop("phi")
        plan = gft.Plan(64, s, d, w, None, phi, dtypes=("f32",), **kw)
        info = plan.info()
        ms = time_kernel(lambda: plan.forward(X, Y, stream), stream, 3, args.table_iters)
        # lane-FMA instructions per signal as generated: dense = n^2, Givens = 2 per rotation +
        # one output multiply per position, exact leaves = sum k^2 (units are adds)
        fmas = 2 * info["n_givens"] + 64 if info["n_givens"] else info["sum_k2"]
        row = {"graph": label, "variant": variant, "adds": info["adds"], "mults": info["mults"],
               "givens": info["n_givens"], "fma_frac": round(fmas * batch / (ms * 1e-3) / fma_peak_per_s("f32"), 4),
               "fast_fwd": {"ms": round(ms, 5), "gbs": round(nbytes / ms / 1e6, 1),
                                                        "frac": round(nbytes / ms / 1e6 / hbm, 4)}}
        if variant == "haar":
            exact[label] = plan.basis()
            msd = time_kernel(lambda: plan.dense_forward(X, Y, stream), stream, 3, args.table_iters)
            rows.append({"graph": label, "variant": "matrix", "adds": info["dense_adds"],
                         "mults": info["dense_mults"], "delta": 0.0, "epsilon": 0.0,
                         "fma_frac": round(4096 * batch / (msd * 1e-3) / fma_peak_per_s("f32"), 4),
                         "fast_fwd": {"ms": round(msd, 5), "gbs": round(nbytes / msd / 1e6, 1),
                                      "frac": round(nbytes / msd / 1e6 / hbm, 4)}})
            row.update(delta=0.0, epsilon=0.0)
        else:
            Uh = plan.basis()
            row.update(delta=round(delta(Uh, exact[label]), 5), epsilon=round(eps(Uh, exact[label]), 5))
        # measured tuning (gft_plan_tune: pacing of FMA-skeleton kernels, the kernel variant of
        # tcgen05 plans), then re-timed
        name0 = plan.kernel_name(0, "f32")
        paces = plan.tune("f32", (0,), X, Y, stream=stream)
        if 0 in paces or plan.kernel_name(0, "f32") != name0:
            ms = time_kernel(lambda: plan.forward(X, Y, stream), stream, 3, args.table_iters)
            row["fast_fwd_tuned"] = {"ms": round(ms, 5), "gbs": round(nbytes / ms / 1e6, 1),
                                     "frac": round(nbytes / ms / 1e6 / hbm, 4), "geometry_pace": paces.get(0),
                                     "kernel": plan.kernel_name(0, "f32")}
        rows.append(row)
        plan.close()
    return rows


def pcie_roof(device):
    """Pinned-host copy bandwidth of this box (256 MiB): H2D, D2H, and each direction while
    both run concurrently -- the roof of the e2e path (one H2D + one D2H per transform)."""
    import torch
    nb = 256 << 20
    hs = torch.empty(nb, dtype=torch.uint8).pin_memory()
    hd = torch.empty(nb, dtype=torch.uint8).pin_memory()
    da = torch.empty(nb, dtype=torch.uint8, device=device)
    db = torch.empty(nb, dtype=torch.uint8, device=device)
    s1, s2 = torch.cuda.Stream(device), torch.cuda.Stream(device)

    def timed(fn, iters=4):
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(iters):
            fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / iters

    def both():
        cur = torch.cuda.current_stream()
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            da.copy_(hs, non_blocking=True)
        with torch.cuda.stream(s2):
            hd.copy_(db, non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)
    out = {"h2d_gbs": round(nb / timed(lambda: da.copy_(hs, non_blocking=True)) / 1e6, 1),
           "d2h_gbs": round(nb / timed(lambda: hd.copy_(db, non_blocking=True)) / 1e6, 1),
           "bidir_each_gbs": round(nb / timed(both) / 1e6, 1)}
    del hs, hd, da, db
    return out


def cpu_oracle_step_time(cfg, X_cpu, budget_s):
    """The oracle (as it stands) on the host: dense fp64 forward + inverse."""
    import oracle
    L = oracle.laplacian(cfg.n, cfg.src, cfg.dst, cfg.w, cfg.self_loops)
    t = time.perf_counter()
    lam, U = oracle.gft_basis(L)
    t_eig = time.perf_counter() - t
    Xn = X_cpu.numpy()
    reps, spent, times = 0, 0.0, []
    while spent < budget_s and reps < 50:
        t = time.perf_counter()
        Y = oracle.forward(Xn, U)
        oracle.inverse(Y, U)
        dt = time.perf_counter() - t
        times.append(dt)
        spent += dt
        reps += 1
    return min(times), statistics.median(times), reps, t_eig


def cpu_oracle_one_thread(cfg, X_cpu):
    """The same oracle step on one BLAS thread (T = nproc and T = 1)."""
    try:
        from threadpoolctl import threadpool_limits
    except Exception:
        return None
    import oracle
    L = oracle.laplacian(cfg.n, cfg.src, cfg.dst, cfg.w, cfg.self_loops)
    lam, U = oracle.gft_basis(L)
    Xn = X_cpu.numpy()
    best = None
    with threadpool_limits(limits=1):
        for _ in range(3):
            t = time.perf_counter()
            oracle.inverse(oracle.forward(Xn, U), U)
            dt = time.perf_counter() - t
            best = dt if best is None else min(best, dt)
    return best


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        return max([i.get("num_threads", 1) for i in threadpool_info()] or [1])
    except Exception:
        return os.cpu_count()


def run_reference(args):
    """--impl reference: the CPU oracle as the reference arm (rank 0 only)."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    import workloads
    cfg = workloads.config(args.config)
    n_ = cfg.n
    rows = min(cfg.batch, args.ref_rows)
    X = workloads.signals(cfg, batch=rows, dtype="f32")
    import oracle
    L = oracle.laplacian(cfg.n, cfg.src, cfg.dst, cfg.w, cfg.self_loops)
    lam, U = oracle.gft_basis(L)
    Xn = X.numpy()
    for _ in range(args.warmup):
        oracle.inverse(oracle.forward(Xn, U), U)
    t = time.perf_counter()
    for _ in range(args.steps):
        oracle.inverse(oracle.forward(Xn, U), U)
    dt = (time.perf_counter() - t) / args.steps
    value = rows / dt
    cores = blas_threads()
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": "signals/s",
           "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic",
           "config": {"workload": "%s: %s" % (args.config, cfg.description), "n": n_,
                      "global_batch": cfg.batch * ws, "per_gpu_batch": cfg.batch,
                      "step": "dense fp64 forward + inverse GFT (the oracle), timed on a bounded "
                              "sample of %d rows per step" % rows,
                      "parallelism": "rank 0 only (CPU)"},
           "cpu_baseline": {"value": value, "unit": "signals/s", "cores": cores, "kind": "oracle",
                            "sample": "%d of %d rows of %s, dense fp64 Y=XU then X=YU^T (numpy BLAS)"
                                      % (rows, cfg.batch, args.config)},
           "e2e": {"value": value, "unit": "signals/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out))
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-table", action="store_true", help="skip the all-config side table")
    ap.add_argument("--table-iters", type=int, default=20)
    ap.add_argument("--no-tune", action="store_true", help="skip the measured-tuning columns of the tables")
    ap.add_argument("--cpu-budget", type=float, default=10.0, help="seconds of oracle CPU timing")
    ap.add_argument("--ref-rows", type=int, default=1 << 20)
    ap.add_argument("--e2e-steps", type=int, default=5)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import workloads
    from paper_1907_07875_b200 import gft

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    dist = None
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=device)
    stream = torch.cuda.current_stream()
    hbm, peak_src = load_peaks()

    cfg = workloads.config(args.config)
    dtype = cfg.dtypes[0]
    t_plan = time.perf_counter()
    plan = gft.Plan.from_config(cfg, dtypes=(dtype,))
    plan.compile(dtype, kinds=(0, 1))   # host plan + kernel load (AOT cubin or NVRTC), reported
    plan_ms = (time.perf_counter() - t_plan) * 1e3
    # weak scaling: every rank transforms its own full batch (seed offset by rank)
    X_cpu = workloads.signals(cfg, dtype=dtype, seed=cfg.seed + rank)
    X = X_cpu.to(device)
    Y = torch.empty_like(X)
    Z = torch.empty_like(X)
    B, n, esz = cfg.batch, cfg.n, X.element_size()

    def step():
        plan.forward(X, Y, stream)
        plan.inverse(Y, Z, stream)

    sampler = ClockSampler(local)
    sampler.start()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier(device)
    torch.cuda.synchronize()
    # timed region: K steps back to back, events only at its ends (an event between two
    # kernels would serialise them and hide the programmatic-dependent-launch overlap)
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    t_start.record(stream)
    for i in range(args.steps):
        plan.forward(X, Y, stream)
        plan.inverse(Y, Z, stream)
    t_end.record(stream)
    torch.cuda.synchronize()
    w1 = time.perf_counter()
    barrier(device)
    sampler.stop()
    total_ms = t_start.elapsed_time(t_end)
    ms_step = max_over_ranks(total_ms / args.steps, device)
    value = B * ws / (ms_step * 1e-3)
    clocks = sampler.summary(w0, w1)
    # per-kernel shares of the step: the same steps again with an event between the kernels
    nsh = max(10, args.steps // 4)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True)) for _ in range(nsh)]
    for i in range(nsh):
        a, b, c = ev[i]
        a.record(stream)
        plan.forward(X, Y, stream)
        b.record(stream)
        plan.inverse(Y, Z, stream)
        c.record(stream)
    torch.cuda.synchronize()
    fwd_all = sorted(ev[i][0].elapsed_time(ev[i][1]) for i in range(nsh))
    inv_all = sorted(ev[i][1].elapsed_time(ev[i][2]) for i in range(nsh))
    fwd_ev = sum(fwd_all) / nsh
    inv_ev = sum(inv_all) / nsh
    # kernel time inside the timed region = step time x the kernel's share of the step
    fwd_ms = ms_step * fwd_ev / (fwd_ev + inv_ev)
    inv_ms = ms_step * inv_ev / (fwd_ev + inv_ev)

    # dominant kernel roofline (algorithmic bytes: read x once + write y once)
    bytes_per_launch = 2 * B * n * esz
    dom_kind, dom_ms = (0, fwd_ms) if fwd_ms >= inv_ms else (1, inv_ms)
    achieved = bytes_per_launch / (dom_ms * 1e-3) / 1e9
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
                "frac": round(achieved / hbm, 4),
                "traffic": load_traffic(KIND_NAMES[dom_kind], args.config, dtype, plan.kernel_name(dom_kind, dtype)),
                "kernel": plan.kernel_name(dom_kind, dtype), "peak_source": peak_src,
                "algorithmic_bytes_per_launch": bytes_per_launch, "avg_launch_ms": round(dom_ms, 5),
                "avg_launch_ms_how": "step time of the timed region x the kernel's share of the step "
                                     "(share from event-bracketed steps, %d)" % nsh,
                "event_bracketed_launch_ms": round(fwd_ev if dom_kind == 0 else inv_ev, 5),
                "nominal_8tbs_frac": round(achieved / 8000.0, 4)}

    # context for the roofline: a plain device copy of the same bytes (torch copy_, read B*n
    # + write B*n) measured the same way -- the best a load+store kernel of this size can do
    copy_ms = time_kernel(lambda: Y.copy_(X), stream, 3, 50)
    roofline["same_size_copy_gbs"] = round(bytes_per_launch / (copy_ms * 1e-3) / 1e9, 1)
    roofline["frac_of_same_size_copy"] = round(achieved / roofline["same_size_copy_gbs"], 4)

    # dense U^T x comparison (same I/O, same stream)
    dense_fwd = time_kernel(lambda: plan.dense_forward(X, Y, stream), stream, 3, 50)
    dense_inv = time_kernel(lambda: plan.dense_inverse(Y, Z, stream), stream, 3, 50)

    # end to end through the C ABI with pinned HOST buffers (H2D + kernel + D2H timed)
    Xh = X_cpu.pin_memory()
    Yh = torch.empty_like(Xh).pin_memory()
    Zh = torch.empty_like(Xh).pin_memory()
    chunk = 1 << 18
    wsb = torch.empty(4 * chunk * n, dtype=X.dtype, device=device)   # 4 slots

    def e2e_step():
        plan.execute_host(0, Xh, Yh, wsb, chunk, stream)
        plan.execute_host(1, Yh, Zh, wsb, chunk, stream)
    for _ in range(3):
        e2e_step()
    torch.cuda.synchronize()
    barrier(device)
    s_e, e_e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s_e.record(stream)
    for _ in range(args.e2e_steps):
        e2e_step()
    e_e.record(stream)
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(s_e.elapsed_time(e_e) / args.e2e_steps, device)
    roundtrip_err = float(((Zh.double() - X_cpu.double()).norm(dim=1) / X_cpu.double().norm(dim=1)).max())
    pcie = pcie_roof(device)
    pcie["achieved_each_dir_gbs"] = round(2 * B * n * esz / (e2e_ms * 1e6), 1)
    pcie["frac_of_bidir"] = round(pcie["achieved_each_dir_gbs"] / pcie["bidir_each_gbs"], 4)

    table = None
    rh_table = ap_table = None
    # the side tables are single-GPU diagnostics; in a multi-rank run the other ranks would
    # only wait for them at the final barrier
    if rank == 0 and not args.no_table and ws == 1:
        table = config_table(args, stream, hbm, device)
        table.append(mixed_cfg5_row(args, stream, hbm, device))
        rh_table = right_haar_table(args, stream, hbm, device)
        ap_table = approx_table(args, stream, hbm, device)

    cpu = None
    if rank == 0:
        best, med, reps, t_eig = cpu_oracle_step_time(cfg, X_cpu, args.cpu_budget)
        cpu = {"value": B / best, "unit": "signals/s", "cores": blas_threads(), "kind": "oracle",
               "sample": "full %s batch (%d x %d), oracle dense fp64 forward+inverse, best of %d "
                         "(median %.3fs); eigensolve %.3fs excluded" % (args.config, B, n, reps, med, t_eig),
               "cpu_model": cpu_model()}
        one = cpu_oracle_one_thread(cfg, X_cpu[: B // 8])
        if one is not None:
            cpu["one_thread_value"] = (B // 8) / one
            cpu["one_thread_sample"] = "first %d rows (1/8 of the batch), same oracle, 1 BLAS thread" % (B // 8)

    if dist:
        dist.barrier()
    if rank == 0:
        info = plan.info()
        out = {
            "metric": METRIC, "value": value, "unit": "signals/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": dtype, "data": "synthetic",
            "config": {"workload": "%s: %s" % (args.config, cfg.description), "n": n,
                       "global_batch": B * ws, "per_gpu_batch": B,
                       "step": "fast forward GFT + fast inverse GFT of the whole batch",
                       "l2": "inputs larger than L2 (%d MiB read+written per launch)" % (bytes_per_launch >> 20),
                       "units_per_level": info["units_per_level"], "leaves": plan.leaf_sizes(),
                       "parallelism": "batch-sharded, no collective" if ws > 1 else "single GPU"},
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": {"value": B * ws / (e2e_ms * 1e-3), "unit": "signals/s",
                    "h2d_bytes_per_step": 2 * B * n * esz, "d2h_bytes_per_step": 2 * B * n * esz,
                    "ms_per_step": e2e_ms, "roundtrip_max_rel_err": roundtrip_err,
                    "path": "gft_execute_host (pinned host; H2D / kernel / D2H stage streams, 4 slots, 2^18-row chunks ramped at both ends)",
                    "pcie": pcie},
            "gpu_launches": 2 * args.steps,
            "kernels": {"fast_fwd_ms": round(fwd_ms, 5), "fast_inv_ms": round(inv_ms, 5),
                        "dense_fwd_ms": round(dense_fwd, 5), "dense_inv_ms": round(dense_inv, 5),
                        "fast_vs_dense": round((dense_fwd + dense_inv) / (fwd_ms + inv_ms), 3),
                        "event_bracketed_fwd_ms_median_min": [round(fwd_all[nsh // 2], 5), round(fwd_all[0], 5)],
                        "event_bracketed_inv_ms_median_min": [round(inv_all[nsh // 2], 5), round(inv_all[0], 5)],
                        "plan_create_and_load_ms": round(plan_ms, 1)},
            "clocks": clocks,
            "configs_table": table,
            "right_haar_table": rh_table,
            "approx_table": ap_table,
        }
        print(json.dumps(out))
    if dist:
        dist.destroy_process_group()
    plan.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
