#!/usr/bin/env python
"""Benchmark of the fused fast-GFT hot path on B200 (contract: DESIGN.md §7).

  python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference] [--tables PATH]

Workload (headline) = BASELINE.json configs[4], the largest single-GPU configuration:
"Mixed large batch" -- the cycle C64 (cfg5a) and the random bipartite N = 128 graph
(cfg5b), 2^20 fp32 signals each.  One step = fast forward + fast inverse GFT of both
batches (rows H1-H6 of SURVEY §8(a), 4 kernel launches); the dense U^T x kernels (H7:
own CUDA-core kernel, a tcgen05 3xTF32 dense kernel and cuBLAS with TF32 off) are timed
beside it on the same inputs -- the paper's comparison "to the GFT realized by a single
n x n matrix multiplication" (§VI-A).

The LAST stdout line is the headline JSON (kept under 2 KiB: the driver reads a bounded
tail).  `--tables PATH` additionally writes the per-config side tables (every BASELINE
config's fast / dense / cuBLAS / filter kernels, right-Haar plans, and the sustained energy
per signal of the headline step vs each dense comparison) to PATH as JSON.
"""
from __future__ import annotations

import argparse
import ctypes
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
WORKLOAD = "cfg5 mixed (configs[4]): C64 (cfg5a) + bipartite N=128 (cfg5b), 2^20 fp32 signals each"


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "MEASURED_PEAKS"
    except Exception:
        return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


def load_traffic(kernel_name):
    """Steady-state DRAM bytes per launch of `kernel_name` from the committed ncu capture
    (profiles/ncu_steady.json: mean of dram__bytes_read+write over launches 2..N of a
    back-to-back sequence with --cache-control none), or None."""
    p = os.path.join(ROOT, "profiles", "ncu_steady.json")
    try:
        with open(p) as f:
            d = json.load(f)
        row = d.get("kernels", {}).get(kernel_name)
        return None if row is None else row.get("dram_bytes_per_launch")
    except Exception:
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
        fn = getattr(self.nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            self.nv.nvmlDeviceGetCurrentClocksThrottleReasons
        while not self._stop.is_set():
            try:
                t = time.perf_counter()
                sm = self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM)
                pw = self.nv.nvmlDeviceGetPowerUsage(self.h) / 1000.0
                self.samples.append((t, sm, fn(self.h), pw))
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

    def energy_mj(self):
        """NVML total energy since driver load (mJ), or None."""
        if not self.ok:
            return None
        try:
            return float(self.nv.nvmlDeviceGetTotalEnergyConsumption(self.h))
        except Exception:
            return None

    def summary(self, t0, t1):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "note": "nvml unavailable"}
        win = [s for s in self.samples if t0 <= s[0] <= t1]
        if not win:   # timed region shorter than the sampling period: nearest samples
            win = sorted(self.samples, key=lambda s: min(abs(s[0] - t0), abs(s[0] - t1)))[:5]
        reasons = set()
        for s in win:
            for bit, name in self.REASONS.items():
                if s[2] & bit and name != "gpu_idle":
                    reasons.add(name)
        return {"sm_mhz": statistics.median([s[1] for s in win]) if win else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(reasons),
                "power_w": round(statistics.median([s[3] for s in win]), 1) if win else None}


from paper_1907_07875_b200.dist import barrier, dist_env, max_over_ranks  # noqa: E402


def measured_compute_peaks(stream):
    """Same-run FFMA / DFMA / tcgen05 kind::tf32 peaks (libgftpeaks.so, best of 3), TFLOP/s."""
    import torch
    from paper_1907_07875_b200 import build as B
    lib = ctypes.CDLL(B.PEAKS_LIB)
    lib.gft_peak_run.restype = ctypes.c_int
    lib.gft_peak_run.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                 ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]
    sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    out = {}
    for which, key in ((0, "ffma_tflops"), (1, "dfma_tflops"), (2, "tf32_tflops"), (3, "ffma_reg_tflops"),
                       (4, "ffma2_tflops")):
        best = 0.0
        for _ in range(3):
            f, ms = ctypes.c_double(), ctypes.c_double()
            rc = lib.gft_peak_run(which, sms, ctypes.c_void_p(stream.cuda_stream), ctypes.byref(f),
                                  ctypes.byref(ms))
            if rc != 0:
                raise RuntimeError("gft_peak_run(%d) failed: cuda error %d" % (which, rc))
            best = max(best, f.value / (ms.value * 1e-3) / 1e12)
        out[key] = round(best, 2)
    # FP32 FMA peak = the faster of the scalar constant-operand and the packed FFMA2 forms
    out["fp32_tflops"] = max(out["ffma_tflops"], out["ffma2_tflops"])
    return out


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


def time_kernel_stats(fn, stream, warmup=5, rounds=5, iters=10):
    """>= 5 warm-up calls, then >= 50 timed calls (rounds x iters back-to-back
    launches, one event pair per round so launches inside a round keep their PDL overlap);
    returns (median, min) of the per-round mean time per call in ms."""
    import torch
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    per = []
    for _ in range(rounds):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        for _ in range(iters):
            fn()
        e.record(stream)
        e.synchronize()
        per.append(s.elapsed_time(e) / iters)
    return statistics.median(per), min(per)


def time_graph(fn, iters):
    """Per-launch device time of `fn` replayed from a captured CUDA graph (launch-bound cases)."""
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


def rec(ms, nbytes, hbm, signals):
    """ms: a time per call, or (median, min) from time_kernel_stats (the median is reported as
    `ms` and feeds every derived figure; `ms_min` beside it)."""
    ms_min = None
    if isinstance(ms, tuple):
        ms, ms_min = ms
    out = {"ms": round(ms, 5), "gbs": round(nbytes / ms / 1e6, 1), "frac": round(nbytes / ms / 1e6 / hbm, 4),
           "signals_per_s": signals / ms * 1e3}
    if ms_min is not None:
        out["ms_min"] = round(ms_min, 5)
    return out


# ------------------------------------------------------------------------------ side tables
def config_table(args, stream, hbm, device, peaks):
    """Every BASELINE config: fast fwd/inv, dense (own CUDA-core, tcgen05, cuBLAS TF32 off)
    and the fused filter, device-resident N(0,1) inputs > L2."""
    import torch
    import workloads
    from paper_1907_07875_b200 import gft
    rows = []

    def tk(fn):   # (median, min) over 5 rounds of max(10, table_iters / 2) calls after 5 warm-up calls
        return time_kernel_stats(fn, stream, 5, 5, max(10, args.table_iters // 2))
    for name, dtype in (("cfg1", "f32"), ("cfg1@2^24", "f32"), ("cfg2", "f32"), ("cfg2b", "f32"),
                        ("cfg3", "f32"), ("cfg4", "f32"), ("cfg4", "f64"), ("cfg5a", "f32"), ("cfg5b", "f32")):
        cfg = workloads.config(name.split("@")[0])
        if "@" in name:   # SURVEY §8(d)'s optional N = 8 bandwidth point (cfg1 itself is launch-bound)
            cfg.batch = 1 << 24
        plan = gft.Plan.from_config(cfg, dtypes=(dtype,))
        tdt = torch.float64 if dtype == "f64" else torch.float32
        g = torch.Generator(device=device).manual_seed(cfg.seed)
        X = torch.randn(cfg.batch, cfg.n, generator=g, device=device, dtype=tdt)
        Y = torch.empty_like(X)
        nbytes = 2 * cfg.batch * cfg.n * X.element_size()
        row = {"config": name, "dtype": dtype, "n": cfg.n, "batch": cfg.batch,
               "units_per_level": plan.info()["units_per_level"], "leaves": plan.leaf_sizes(),
               "kernel_fwd": plan.kernel_name(0, dtype), "kernel_dense_fwd": plan.kernel_name(2, dtype)}
        for kind, f in ((0, plan.forward), (1, plan.inverse), (2, plan.dense_forward), (3, plan.dense_inverse)):
            row[KIND_NAMES[kind]] = rec(tk(lambda: f(X, Y, stream)), nbytes, hbm, cfg.batch)
        if cfg.batch * cfg.n * X.element_size() <= (64 << 20):   # launch-bound: replay a graph
            row["fast_fwd"]["graph_ms"] = round(time_graph(lambda: plan.forward(X, Y), 50), 5)
            Z1 = torch.empty_like(X)
            row["fwd_inv_pair_graph_ms"] = round(time_graph(lambda: (plan.forward(X, Y), plan.inverse(Y, Z1)), 50), 5)
        pk = peaks["fp32_tflops" if dtype == "f32" else "dfma_tflops"] * 1e12
        row["dense_fwd"]["fma_frac"] = round(2.0 * cfg.n * cfg.n * cfg.batch / (row["dense_fwd"]["ms"] * 1e-3) / pk, 4)
        row["fast_vs_dense_fwd"] = round(row["dense_fwd"]["ms"] / row["fast_fwd"]["ms"], 3)
        filt = gft.Filter(plan, np.exp(-plan.eigenvalues()), dtypes=(dtype,))
        row["filter"] = dict(rec(tk(lambda: filt.apply(X, Y, stream)), nbytes, hbm, cfg.batch), kernel=filt.kernel_name(dtype))
        row["fused_filter_vs_two_pass"] = round((row["fast_fwd"]["ms"] + row["fast_inv"]["ms"]) / row["filter"]["ms"], 3)
        U = torch.from_numpy(plan.basis()).to(device=device, dtype=tdt)
        tf32 = torch.backends.cuda.matmul.allow_tf32
        torch.backends.cuda.matmul.allow_tf32 = False
        row["cublas_fwd"] = rec(tk(lambda: torch.matmul(X, U, out=Y)), nbytes, hbm, cfg.batch)
        torch.backends.cuda.matmul.allow_tf32 = tf32
        best = min(row["dense_fwd"]["ms"], row["cublas_fwd"]["ms"])
        if dtype == "f32" and cfg.n % 32 == 0:
            dplan = gft.Plan.from_config(cfg, dtypes=(dtype,), dense_tc=True)
            row["dense_tc_fwd"] = dict(rec(tk(lambda: dplan.dense_forward(X, Y, stream)), nbytes, hbm, cfg.batch),
                                       kernel=dplan.kernel_name(2, dtype))
            best = min(best, row["dense_tc_fwd"]["ms"])
            dplan.close()
        row["fast_vs_best_dense_fwd"] = round(best / row["fast_fwd"]["ms"], 3)
        if args.tune and cfg.batch * cfg.n * X.element_size() > (64 << 20):
            ch = plan.tune(dtype, (0, 1), X, Y, stream=stream, geometry=True)
            for kind, f in ((0, plan.forward), (1, plan.inverse)):
                if kind in ch:
                    row[KIND_NAMES[kind] + "_tuned"] = dict(rec(tk(lambda: f(X, Y, stream)), nbytes, hbm, cfg.batch),
                                                            geometry_pace=ch[kind])
        rows.append(row)
        del X, Y
        filt.close()
        plan.close()
    return rows


def paper_table(args, stream, hbm, device):
    """tab:runtime of Sec. VI-A re-timed on B200: the paper's graphs, its
    printed operation counts and C-runtime reductions (hardware not stated) beside ours.
    Signals are i.i.d. U[0,1] fp32 as in PAPER.md:757, at the paper's 20000 signals (launch-
    bound: CUDA-graph replay) and at 2^21 (bandwidth regime).  runtime reduction =
    1 - t_fast / t_dense for the forward transform, against our CUDA-core dense kernel (the
    "single n x n matrix multiplication" analogue) and against the best dense kernel."""
    import torch
    import workloads
    from paper_1907_07875_b200 import gft
    rows = []
    tf32 = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    for topo, n, build, phi, paper_ops, paper_red in workloads.tab_runtime_graphs():
        s, d, w = build()
        plan = gft.Plan(n, s, d, w, None, phi, dtypes=("f32",))
        info = plan.info()
        row = {"topology": topo, "n": n, "leaves": plan.leaf_sizes(),
               "paper": {"matrix_adds": paper_ops[0], "matrix_mults": paper_ops[1], "fast_adds": paper_ops[2],
                         "fast_mults": paper_ops[3], "runtime_reduction_pct": paper_red,
                         "hardware": "not stated (C implementation)"},
               "ours": {"fast_adds": info["adds"], "fast_mults_paper_convention": info["paper_mults"],
                        "fast_mults_kernel": info["mults"]}}
        # tcgen05 dense comparison wherever the tensor-core kernels apply (n % 4 == 0, rows padded
        # to 32 columns) and the product is big enough to matter
        dplan = gft.Plan(n, s, d, w, None, phi, dtypes=("f32",), dense_tc=True) if n % 4 == 0 and n >= 32 else None
        U = torch.from_numpy(plan.basis()).to(device=device, dtype=torch.float32)
        for batch in (20000, 1 << 21):
            g = torch.Generator(device=device).manual_seed(n)
            X = torch.rand(batch, n, generator=g, device=device)
            Y = torch.empty_like(X)
            # current stream (= `stream`), so that the same calls can be captured into a graph
            arms = {"fast": lambda: plan.forward(X, Y), "dense": lambda: plan.dense_forward(X, Y),
                    "cublas": lambda: torch.matmul(X, U, out=Y)}
            if dplan is not None:
                arms["dense_tc"] = lambda: dplan.dense_forward(X, Y)
            if batch <= 20000:
                t = {k: time_graph(f, 50) for k, f in arms.items()}
            else:
                t = {k: time_kernel(f, stream, 3, args.table_iters) for k, f in arms.items()}
            best = min(v for k, v in t.items() if k != "fast")
            row["b%d" % batch] = {"ms": {k: round(v, 5) for k, v in t.items()},
                                  "reduction_vs_dense_pct": round(100 * (1 - t["fast"] / t["dense"]), 1),
                                  "reduction_vs_best_dense_pct": round(100 * (1 - t["fast"] / best), 1),
                                  "fast_hbm_frac": round(2 * batch * n * 4 / (t["fast"] * 1e-3) / 1e9 / hbm, 4)}
            del X, Y
        rows.append(row)
        if dplan is not None:
            dplan.close()
        plan.close()
    torch.backends.cuda.matmul.allow_tf32 = tf32
    return rows


def energy_config_table(stream, sampler, seconds, device):
    """Per-config energy: the fast forward against each dense forward of the same config (own
    CUDA-core kernel, tcgen05 dense where it applies, cuBLAS TF32 off), each back to back for
    `seconds` at the power cap, on the configs where the dense product is not trivially
    HBM-bound (n = 64 / 128, fp32 and fp64)."""
    import torch
    import workloads
    from paper_1907_07875_b200 import gft
    out = []
    for name, dtype in (("cfg4", "f32"), ("cfg4", "f64"), ("cfg5a", "f32"), ("cfg5b", "f32")):
        cfg = workloads.config(name)
        plan = gft.Plan.from_config(cfg, dtypes=(dtype,))
        tdt = torch.float64 if dtype == "f64" else torch.float32
        X = torch.randn(cfg.batch, cfg.n, generator=torch.Generator(device=device).manual_seed(cfg.seed),
                        device=device, dtype=tdt)
        Y = torch.empty_like(X)
        U = torch.from_numpy(plan.basis()).to(device=device, dtype=tdt)
        arms = {"fast": lambda: plan.forward(X, Y, stream), "dense": lambda: plan.dense_forward(X, Y, stream),
                "cublas": lambda: torch.matmul(X, U, out=Y)}
        dplan = None
        if dtype == "f32":
            dplan = gft.Plan.from_config(cfg, dtypes=(dtype,), dense_tc=True)
            arms["dense_tc"] = lambda: dplan.dense_forward(X, Y, stream)
        arms["copy"] = lambda: Y.copy_(X)
        rows = energy_table(arms, cfg.batch, stream, sampler, seconds, bytes_per_step=2 * X.numel() * X.element_size())
        out.append({"config": name, "dtype": dtype, "arms": rows})
        if dplan is not None:
            dplan.close()
        plan.close()
        del X, Y
    return out


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def oracle_table(max_rows):
    """SURVEY §8(d) oracle timing: the oracle's dense fp64 forward Y = X U of every config on
    the host, with all BLAS threads and with 1 thread (bounded to `max_rows` rows per config)."""
    import oracle
    import workloads
    try:
        from threadpoolctl import threadpool_limits
    except ImportError:   # pragma: no cover
        threadpool_limits = None
    out = {"cpu_model": cpu_model(), "cores": os.cpu_count(), "blas_threads": blas_threads(), "configs": []}
    for name, dtype in (("cfg2", "f32"), ("cfg3", "f32"), ("cfg4", "f32"), ("cfg4", "f64"), ("cfg5a", "f32"),
                        ("cfg5b", "f32")):
        cfg = workloads.config(name)
        rows = min(cfg.batch, max_rows)
        U = oracle.gft_basis(oracle.laplacian(cfg.n, cfg.src, cfg.dst, cfg.w, cfg.self_loops))[1]
        X = workloads.signals(cfg, batch=rows, dtype=dtype).numpy()
        r = {"config": name, "dtype": dtype, "rows": rows}
        for tag, nt in (("all_threads", None), ("one_thread", 1)):
            ctx = threadpool_limits(limits=nt) if (threadpool_limits and nt) else None
            if ctx:
                ctx.__enter__()
            try:
                best = 1e9
                for _ in range(2):
                    t = time.perf_counter()
                    oracle.forward(X, U)
                    best = min(best, time.perf_counter() - t)
            finally:
                if ctx:
                    ctx.__exit__(None, None, None)
            r[tag + "_signals_per_s"] = rows / best
        out["configs"].append(r)
    return out


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
        X = torch.randn(batch, n, generator=torch.Generator(device=device).manual_seed(5), device=device, dtype=tdt)
        Y = torch.empty_like(X)
        nbytes = 2 * batch * n * X.element_size()
        row = {"graph": label, "dtype": dtype, "n": n, "batch": batch}
        for tag, rh in (("right_haar", True), ("one_block", False)):
            plan = gft.Plan(n, s, d, w, loops, dtypes=(dtype,), normalized=norm, right_haar=rh)
            info = plan.info()
            r = {"leaves": plan.leaf_sizes(), "pairs": info["n_right_pairs"], "mults": info["mults"],
                 "adds": info["adds"], "kernel": plan.kernel_name(0, dtype)}
            for k, f in ((0, plan.forward), (1, plan.inverse)):
                r[KIND_NAMES[k]] = rec(time_kernel_stats(lambda: f(X, Y, stream), stream, 5, 5, max(10, args.table_iters // 2)),
                                       nbytes, hbm, batch)
            row[tag] = r
            plan.close()
        row["right_vs_one_block_fwd"] = round(row["one_block"]["fast_fwd"]["ms"] / row["right_haar"]["fast_fwd"]["ms"], 3)
        rows.append(row)
        del X, Y
    return rows


def energy_table(arms, signals_per_step, stream, sampler, seconds, bytes_per_step=None):
    """Sustained throughput and energy per signal of the headline step (fast GFT) against the
    dense U^T x comparisons on the same inputs, each run back to back for `seconds` at the
    power cap (the paper's premise: one graph, many transforms).  Energy from
    NVML's total-energy counter around each window; the fast arm runs first and last (drift)."""
    import torch
    rows = []
    order = list(arms) + [list(arms)[0]]
    for name in order:
        fn = arms[name]
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0 = sampler.energy_mj()
        w0 = time.perf_counter()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        n, tot = 0, 0.0
        while tot < seconds * 1e3:
            for _ in range(20):
                fn()
            n += 20
            b.record(stream)
            b.synchronize()
            tot = a.elapsed_time(b)
        w1 = time.perf_counter()
        e1 = sampler.energy_mj()
        c = sampler.summary(w0, w1)
        ms = tot / n
        row = {"arm": name, "seconds": round(tot / 1e3, 2), "ms_per_step": round(ms, 5),
               "signals_per_s": signals_per_step / (ms * 1e-3), "sm_mhz": c["sm_mhz"], "power_w": c["power_w"],
               "reasons": c["reasons"]}
        if e0 is not None and e1 is not None:
            row["avg_power_w"] = round((e1 - e0) / 1e3 / (w1 - w0), 1)
            row["nj_per_signal"] = round((e1 - e0) * 1e6 / (n * signals_per_step), 3)
            if bytes_per_step:
                row["pj_per_byte"] = round((e1 - e0) * 1e9 / (n * bytes_per_step), 1)
        rows.append(row)
    return rows


# ------------------------------------------------------------------------------ helpers
def _round_sig(v, sig=6):
    if isinstance(v, float):
        return float("%.*g" % (sig, v))
    if isinstance(v, dict):
        return {k: _round_sig(x, sig) for k, x in v.items()}
    if isinstance(v, list):
        return [_round_sig(x, sig) for x in v]
    return v


def headline_line(out, limit=2000):
    """The last stdout line: floats to 6 significant digits (the top-level value and
    ms_per_step keep full precision), then -- only if still over `limit` bytes, so that the
    line survives a bounded stdout tail -- the least important keys are dropped in order."""
    top = {k: out[k] for k in ("value", "ms_per_step") if k in out}
    out = _round_sig(out)
    out.update(top)
    line = json.dumps(out, separators=(",", ":"))
    for path in (("peaks_tflops",), ("kernels", "share"), ("cpu_baseline", "sample"), ("kernels",)):
        if len(line) <= limit:
            break
        d = out
        for k in path[:-1]:
            d = d.get(k, {})
        d.pop(path[-1], None)
        line = json.dumps(out, separators=(",", ":"))
    return line


def pcie_roof(device):
    """Pinned-host copy bandwidth of this box (256 MiB), each direction while both run
    concurrently -- the roof of the e2e path."""
    import torch
    nb = 256 << 20
    hs = torch.empty(nb, dtype=torch.uint8).pin_memory()
    hd = torch.empty(nb, dtype=torch.uint8).pin_memory()
    da = torch.empty(nb, dtype=torch.uint8, device=device)
    db = torch.empty(nb, dtype=torch.uint8, device=device)
    s1, s2 = torch.cuda.Stream(device), torch.cuda.Stream(device)

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
    both()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(4):
        both()
    b.record()
    torch.cuda.synchronize()
    out = round(nb / (a.elapsed_time(b) / 4) / 1e6, 1)
    del hs, hd, da, db
    return out


def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        return max([i.get("num_threads", 1) for i in threadpool_info()] or [1])
    except Exception:
        return os.cpu_count()


def oracle_mixed_step(cfgs, rows, budget_s=None, steps=None, warmup=0):
    """The oracle (as it stands) on the host: dense fp64 forward + inverse of `rows` signals
    of each graph of the mixed workload.  Returns (seconds per step, #signals, reps)."""
    import oracle
    import workloads
    mats, data = [], []
    for cfg in cfgs:
        L = oracle.laplacian(cfg.n, cfg.src, cfg.dst, cfg.w, cfg.self_loops)
        mats.append(oracle.gft_basis(L)[1])
        data.append(workloads.signals(cfg, batch=rows, dtype="f32").numpy())

    def one():
        for U, X in zip(mats, data):
            oracle.inverse(oracle.forward(X, U), U)
    for _ in range(warmup):
        one()
    times = []
    t_all = time.perf_counter()
    while True:
        t = time.perf_counter()
        one()
        times.append(time.perf_counter() - t)
        if steps is not None and len(times) >= steps:
            break
        if steps is None and (time.perf_counter() - t_all >= budget_s or len(times) >= 50):
            break
    return times, rows * len(cfgs)


def run_reference(args):
    """--impl reference: the CPU oracle as the reference arm (rank 0 only)."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    import workloads
    cfgs = [workloads.config("cfg5a"), workloads.config("cfg5b")]
    times, sig = oracle_mixed_step(cfgs, args.ref_rows, steps=args.steps, warmup=args.warmup)
    dt = sum(times) / len(times)
    value = sig / dt
    sample = ("%d of 2^20 rows of each of cfg5a and cfg5b per step, oracle dense fp64 Y=XU then X=YU^T "
              "(numpy BLAS)" % args.ref_rows)
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": "signals/s", "n_gpus": ws,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": WORKLOAD, "global_batch": 2 << 20, "per_gpu_batch": 2 << 20,
                      "step": "dense fp64 forward + inverse of both graphs (the oracle), bounded sample",
                      "parallelism": "rank 0 only (CPU)"},
           "cpu_baseline": {"value": value, "unit": "signals/s", "cores": blas_threads(), "kind": "oracle",
                            "sample": sample},
           "e2e": {"value": value, "unit": "signals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))
    return 0


# ------------------------------------------------------------------------------ main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--tables", default=None, help="write the per-config side tables (JSON) to this path")
    ap.add_argument("--table-iters", type=int, default=20)
    ap.add_argument("--tune", action="store_true", help="measured-tuning columns in the side tables")
    ap.add_argument("--sustain-s", type=float, default=2.0, help="seconds of the sustained-load arm (0: skip)")
    ap.add_argument("--cpu-budget", type=float, default=10.0, help="seconds of oracle CPU timing")
    ap.add_argument("--ref-rows", type=int, default=1 << 17, help="oracle sample rows per graph")
    ap.add_argument("--e2e-steps", type=int, default=2, help="steps per e2e round")
    ap.add_argument("--e2e-rounds", type=int, default=5, help="e2e rounds (the median is reported)")
    ap.add_argument("--energy-s", type=float, default=2.0, help="seconds per arm of the energy side table")
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

    # ---- the mixed workload: cfg5a (C64) + cfg5b (bipartite N = 128), fp32 -----------------
    cfgs = [workloads.config("cfg5a"), workloads.config("cfg5b")]
    t0 = time.perf_counter()
    plans = [gft.Plan.from_config(c, dtypes=("f32",)) for c in cfgs]
    for p in plans:
        p.compile("f32", kinds=(0, 1, 2, 3))
    plan_ms = (time.perf_counter() - t0) * 1e3
    # weak scaling: every rank transforms its own full batches (seed offset by rank)
    Xc = [workloads.signals(c, dtype="f32", seed=c.seed + rank) for c in cfgs]
    X = [x.to(device) for x in Xc]
    Y = [torch.empty_like(x) for x in X]
    Z = [torch.empty_like(x) for x in X]
    B = sum(c.batch for c in cfgs)
    nbytes = [2 * c.batch * c.n * 4 for c in cfgs]   # algorithmic bytes per launch (read x + write y)
    # launch order of one step; (plan index, kind)
    seq = [(0, 0), (1, 0), (0, 1), (1, 1)]

    def launch(i, kind):
        if kind == 0:
            plans[i].forward(X[i], Y[i], stream)
        else:
            plans[i].inverse(Y[i], Z[i], stream)

    def step():
        for i, k in seq:
            launch(i, k)

    sampler = ClockSampler(local)
    sampler.start()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier(device)
    torch.cuda.synchronize()
    # timed region: K steps back to back, events only at its ends (an event between two
    # kernels would serialise them and hide the programmatic-dependent-launch overlap)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    ev0.record(stream)
    for _ in range(args.steps):
        step()
    ev1.record(stream)
    torch.cuda.synchronize()
    w1 = time.perf_counter()
    barrier(device)
    ms_step = max_over_ranks(ev0.elapsed_time(ev1) / args.steps, device)
    value = B * ws / (ms_step * 1e-3)
    clocks = sampler.summary(w0, w1)

    # per-kernel shares: the same steps again with an event between every launch
    nsh = max(20, args.steps)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(len(seq) + 1)] for _ in range(nsh)]
    for r in range(nsh):
        evs[r][0].record(stream)
        for j, (i, k) in enumerate(seq):
            launch(i, k)
            evs[r][j + 1].record(stream)
    torch.cuda.synchronize()
    per = [sum(evs[r][j].elapsed_time(evs[r][j + 1]) for r in range(nsh)) / nsh for j in range(len(seq))]
    share = [p / sum(per) for p in per]
    dom = max(range(len(seq)), key=lambda j: per[j])
    di, dk = seq[dom]
    dom_ms = ms_step * share[dom]        # the dominant kernel's time inside the timed region
    dname = plans[di].kernel_name(dk, "f32")
    achieved = nbytes[di] / (dom_ms * 1e-3) / 1e9

    # ---- same-run compute peaks (FFMA, DFMA, tcgen05 TF32) --------------------------------
    peaks = measured_compute_peaks(stream)
    # the dominant kernel's tensor-pipe load: 3xTF32 = 3 MMA passes over each tensor-core leaf
    info = plans[di].info()
    tc_flops = 3 * 2.0 * info["sum_k2"] * cfgs[di].batch if "tc" in dname else 0.0
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
                "frac": round(achieved / hbm, 4), "traffic": load_traffic(dname), "kernel": dname,
                "peak_src": peak_src, "bytes_per_launch": nbytes[di], "launch_ms": round(dom_ms, 5),
                "event_bracketed_ms": round(per[dom], 5),
                "tensor_frac": round(tc_flops / (dom_ms * 1e-3) / (peaks["tf32_tflops"] * 1e12), 4)}

    # ---- the in-run dense U^T x comparisons (same inputs, fwd + inv of both per step) ------
    def dense_step_ms(fwd, inv):
        def f():
            for i in range(2):
                fwd(i)
                inv(i)
        return time_kernel(f, stream, 3, 10)
    dense = {}
    dense["fma"] = dense_step_ms(lambda i: plans[i].dense_forward(X[i], Y[i], stream),
                                     lambda i: plans[i].dense_inverse(Y[i], Z[i], stream))
    dplans = [gft.Plan.from_config(c, dtypes=("f32",), dense_tc=True) for c in cfgs]
    dense["tc"] = dense_step_ms(lambda i: dplans[i].dense_forward(X[i], Y[i], stream),
                                     lambda i: dplans[i].dense_inverse(Y[i], Z[i], stream))
    Us = [torch.from_numpy(p.basis()).to(device=device, dtype=torch.float32) for p in plans]
    tf32 = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    dense["cublas"] = dense_step_ms(lambda i: torch.matmul(X[i], Us[i], out=Y[i]),
                                    lambda i: torch.matmul(Y[i], Us[i].t(), out=Z[i]))
    torch.backends.cuda.matmul.allow_tf32 = tf32
    dense_flops = sum(2 * 2.0 * c.n * c.n * c.batch for c in cfgs)   # fwd + inv, both graphs
    kernels = {"fast_ms_per_step": round(ms_step, 5),
               "share": {"%s_%s" % (cfgs[i].name[3:], "fwd" if k == 0 else "inv"): round(share[j], 3)
                         for j, (i, k) in enumerate(seq)},
               "dense_ms_per_step": {k: round(v, 5) for k, v in dense.items()},
               "fast_vs_dense": {k: round(v / ms_step, 3) for k, v in dense.items()},
               "fast_vs_best_dense": round(min(dense.values()) / ms_step, 3),
               "fma_dense_frac": round(dense_flops / (dense["fma"] * 1e-3) / (peaks["fp32_tflops"] * 1e12), 4),
               "plan_create_and_load_ms": round(plan_ms, 1)}

    # ---- side tables (file only) ----------------------------------------------------------
    if args.tables and rank == 0 and ws == 1:
        arms = {"fast": step,
                "dense_tc": lambda: [(dplans[i].dense_forward(X[i], Y[i], stream),
                                      dplans[i].dense_inverse(Y[i], Z[i], stream)) for i in range(2)],
                "dense_fma": lambda: [(plans[i].dense_forward(X[i], Y[i], stream),
                                       plans[i].dense_inverse(Y[i], Z[i], stream)) for i in range(2)],
                "cublas_tf32_off": lambda: [(torch.matmul(X[i], Us[i], out=Y[i]),
                                             torch.matmul(Y[i], Us[i].t(), out=Z[i])) for i in range(2)],
                # the same bytes moved by plain device copies: the data-movement energy floor
                "copy": lambda: [(Y[i].copy_(X[i]), Z[i].copy_(Y[i])) for i in range(2)]}
        tf32 = torch.backends.cuda.matmul.allow_tf32
        torch.backends.cuda.matmul.allow_tf32 = False
        tables = {"hbm_peak_gbs": hbm, "compute_peaks": peaks,
                  "energy": energy_table(arms, B, stream, sampler, args.energy_s, bytes_per_step=2 * sum(nbytes)),
                  "energy_configs": energy_config_table(stream, sampler, 0.5 * args.energy_s, device),
                  "configs": config_table(args, stream, hbm, device, peaks),
                  "right_haar": right_haar_table(args, stream, hbm, device),
                  "paper_tab_runtime": paper_table(args, stream, hbm, device),
                  "oracle_cpu": oracle_table(1 << 18)}
        torch.backends.cuda.matmul.allow_tf32 = tf32
        os.makedirs(os.path.dirname(os.path.abspath(args.tables)), exist_ok=True)
        with open(args.tables, "w") as f:
            json.dump(tables, f, indent=1)

    # ---- sustained load: >= sustain_s seconds of back-to-back steps at the power cap (after
    # the dense comparisons: a hot GPU sits at a capped clock for a while), then the same for
    # the tcgen05 dense step -- the fast transform's fewer operations show as energy per signal
    # and as a higher capped clock (one graph, many transforms) -----------------
    sustained = None
    if args.sustain_s > 0:
        def sustain(fn, ms_hint):
            chunk = max(1, int(200.0 / ms_hint))   # ~0.2 s of steps per event pair
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            tot_ms, nsteps = 0.0, 0
            e0 = sampler.energy_mj()
            s0 = time.perf_counter()
            a.record(stream)
            while tot_ms < args.sustain_s * 1e3:
                for _ in range(chunk):
                    fn()
                nsteps += chunk
                b.record(stream)
                b.synchronize()
                tot_ms = a.elapsed_time(b)
            s1 = time.perf_counter()
            e1 = sampler.energy_mj()
            sms = max_over_ranks(tot_ms / nsteps, device)
            nj = None if e0 is None or e1 is None else round((e1 - e0) * 1e6 / (nsteps * B), 1)
            return tot_ms, sms, sampler.summary(s0, s1), nj
        tot_ms, sms, sc, nj = sustain(step, ms_step)
        sustained = {"seconds": round(tot_ms / 1e3, 2), "ms_per_step": round(sms, 5),
                     "value": B * ws / (sms * 1e-3),
                     "dominant_frac": round(nbytes[di] / (sms * share[dom] * 1e-3) / 1e9 / hbm, 4),
                     "nj_per_signal": nj,
                     "clocks": {k: sc[k] for k in ("sm_mhz", "reasons", "power_w")}}
        tc_step = lambda: [(dplans[i].dense_forward(X[i], Y[i], stream),   # noqa: E731
                            dplans[i].dense_inverse(Y[i], Z[i], stream)) for i in range(2)]
        _, tms, tsc, tnj = sustain(tc_step, dense["tc"])
        sustained["dense_tc"] = {"ms_per_step": round(tms, 5), "fast_speedup": round(tms / sms, 3),
                                 "nj_per_signal": tnj, "sm_mhz": tsc["sm_mhz"]}
        # the same bytes as plain device copies: what the box sustains for pure data movement
        copy_step = lambda: [(Y[i].copy_(X[i]), Z[i].copy_(Y[i])) for i in range(2)]   # noqa: E731
        _, cms, _, cnj = sustain(copy_step, ms_step)
        sustained["copy"] = {"ms_per_step": round(cms, 5), "fast_frac_of_copy": round(cms / sms, 4),
                             "nj_per_signal": cnj}
    for p in dplans:
        p.close()
    sampler.stop()

    # ---- end to end through the C ABI with pinned HOST buffers (H2D + kernels + D2H timed) ---
    Xh = [x.pin_memory() for x in Xc]
    Yh = [torch.empty_like(x).pin_memory() for x in Xh]
    Zh = [torch.empty_like(x).pin_memory() for x in Xh]
    chunk_rows = 1 << 17
    wsb = [torch.empty(4 * chunk_rows * c.n, dtype=torch.float32, device=device) for c in cfgs]

    # one caller stream per graph: the two graphs' transfers pipeline back to back through the
    # library's shared H2D / kernel / D2H stage streams (no drain bubble between calls); each
    # graph's inverse still follows its forward (stream order on its own stream)
    gstreams = [torch.cuda.Stream(device), torch.cuda.Stream(device)]

    def e2e_step():
        for s in gstreams:
            s.wait_stream(stream)
        for d in (0, 1):
            for i in range(2):
                plans[i].execute_host(d, Xh[i] if d == 0 else Yh[i], Yh[i] if d == 0 else Zh[i], wsb[i], chunk_rows,
                                      gstreams[i])
        for s in gstreams:
            stream.wait_stream(s)
    e2e_step()
    torch.cuda.synchronize()
    barrier(device)
    # median over rounds of e2e_steps steps each (one round on a box once read 0.73 of the
    # PCIe roof where every other run, before and after, read 0.96-0.98: tools/r02/e2e_var.py)
    rounds = []
    for _ in range(args.e2e_rounds):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(args.e2e_steps):
            e2e_step()
        b.record(stream)
        torch.cuda.synchronize()
        rounds.append(a.elapsed_time(b) / args.e2e_steps)
    e2e_ms = max_over_ranks(statistics.median(rounds), device)
    rt_err = max(float(((z.double() - x.double()).norm(dim=1) / x.double().norm(dim=1)).max())
                 for z, x in zip(Zh, Xc))
    step_bytes = sum(nbytes)   # per step: each transform copies its input in and its output out
    e2e = {"value": B * ws / (e2e_ms * 1e-3), "unit": "signals/s", "h2d_bytes_per_step": step_bytes,
           "d2h_bytes_per_step": step_bytes, "ms_per_step": round(e2e_ms, 4), "rounds": "median of %d x %d steps" % (args.e2e_rounds, args.e2e_steps),
           "roundtrip_max_rel_err": rt_err,
           "pcie_bidir_each_gbs": pcie_roof(device),
           "achieved_each_dir_gbs": round(step_bytes / (e2e_ms * 1e6), 1)}

    cpu = None
    if rank == 0:
        times, sig = oracle_mixed_step(cfgs, args.ref_rows, budget_s=args.cpu_budget)
        cpu = {"value": sig / min(times), "unit": "signals/s", "cores": blas_threads(), "kind": "oracle",
               "sample": "%d rows of each of cfg5a and cfg5b, oracle dense fp64 fwd+inv, best of %d"
                         % (args.ref_rows, len(times))}

    if dist:
        dist.barrier()
    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": "signals/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": WORKLOAD, "global_batch": B * ws, "per_gpu_batch": B,
                       "step": "fast fwd + fast inv of both batches (4 launches)",
                       "l2": "inputs > L2 (768 MiB in + out per step)",
                       "parallelism": "batch-sharded replicas, no collective" if ws > 1 else "single GPU"},
            "roofline": roofline, "peaks_tflops": peaks, "sustained": sustained,
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": len(seq) * args.steps,
            "kernels": kernels, "clocks": clocks,
        }
        print(headline_line(out), flush=True)
    if dist:
        dist.destroy_process_group()
    for p in plans:
        p.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
