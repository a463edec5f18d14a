"""Build the C-ABI library (and the AOT cubin cache of the BASELINE configs).

  python -m paper_1907_07875_b200.build            # libgft.so + AOT cubins
  python -m paper_1907_07875_b200.build --no-aot   # library only

The library (host planner + codegen + driver runtime) is compiled with g++ and has no
link-time dependency on libcuda / libnvrtc (both are dlopen-ed), so it loads on a
CPU-only host.  The AOT step generates the plan-specialised kernels of the BASELINE
configurations through the library itself and compiles each with
`nvcc -cubin -gencode arch=compute_100a,code=sm_100a -lineinfo`, storing them under
_lib/kernels/<kernel-name>.cubin where the runtime finds them before falling back to
NVRTC.  The kernel name embeds a hash of the full generated source, so a stale cubin
can never be picked up for a different plan.
"""
from __future__ import annotations

import argparse
import hashlib
import os
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "_lib")
LIB = os.path.join(LIBDIR, "libgft.so")
KDIR = os.path.join(LIBDIR, "kernels")
CUDA_HOME = os.environ.get("CUDA_HOME", "/usr/local/cuda")
SOURCES = ["plan.cpp", "search.cpp", "codegen.cpp", "cuda_rt.cpp", "capi.cpp", "serialize.cpp"]
ARCH = "-gencode=arch=compute_100a,code=sm_100a"


SKELETONS = {"kernel_skeleton.cuh": "skeleton_inc.h", "kernel_tc_skeleton.cuh": "skeleton_tc_inc.h",
             "kernel_tc2_skeleton.cuh": "skeleton_tc2_inc.h", "kernel_tc3_skeleton.cuh": "skeleton_tc3_inc.h",
             "kernel_dense_skeleton.cuh": "skeleton_dense_inc.h"}


def _write_skeleton_inc():
    for src, dst in SKELETONS.items():
        with open(os.path.join(CSRC, src)) as f:
            text = f.read()
        assert ")GFTSKEL\"" not in text
        out = os.path.join(CSRC, dst)
        new = 'R"GFTSKEL(' + text + ')GFTSKEL"\n'
        if not os.path.exists(out) or open(out).read() != new:
            with open(out, "w") as f:
                f.write(new)


def _stamp():
    h = hashlib.sha256()
    for s in SOURCES + ["plan.hpp", "kernels.hpp"] + list(SKELETONS):
        with open(os.path.join(CSRC, s), "rb") as f:
            h.update(f.read())
    with open(os.path.join(ROOT, "include", "gft.h"), "rb") as f:
        h.update(f.read())
    return h.hexdigest()


def build_library(force=False, verbose=True):
    os.makedirs(LIBDIR, exist_ok=True)
    _write_skeleton_inc()
    stamp = _stamp()
    stamp_file = LIB + ".stamp"
    if not force and os.path.exists(LIB) and os.path.exists(stamp_file) and open(stamp_file).read() == stamp:
        return LIB
    objs = []
    with tempfile.TemporaryDirectory() as td:
        procs = []
        for s in SOURCES:
            o = os.path.join(td, s + ".o")
            cmd = ["g++", "-std=c++17", "-O2", "-g", "-fPIC", "-Wall", "-Wno-unused-function",
                   "-fvisibility=hidden", "-I", os.path.join(CUDA_HOME, "include"),
                   "-I", os.path.join(ROOT, "include"), "-c", os.path.join(CSRC, s), "-o", o]
            procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
            objs.append(o)
        for cmd, p in procs:
            out = p.communicate()[0].decode()
            if p.returncode != 0:
                raise RuntimeError("compile failed: " + " ".join(cmd) + "\n" + out)
            if verbose and out.strip():
                print(out)
        tmp = LIB + ".tmp"
        cmd = ["g++", "-shared", "-o", tmp] + objs + ["-ldl", "-lpthread"]
        subprocess.check_call(cmd)
        os.replace(tmp, LIB)
    with open(stamp_file, "w") as f:
        f.write(stamp)
    if verbose:
        print("built", LIB)
    return LIB


def aot_kernel_specs():
    """(config name, dtype list, plan kwargs) of the kernels shipped as AOT cubins."""
    import workloads
    specs = []
    for name in ("cfg1", "cfg2", "cfg2b", "cfg3", "cfg4", "cfg5a", "cfg5b"):
        cfg = workloads.config(name)
        depths = [cfg.max_depth] + ([1] if name == "cfg1" else [])
        for md in depths:
            specs.append((cfg, list(cfg.dtypes), md))
    return specs


def build_aot_cubins(jobs=8, verbose=True):
    """Generate the BASELINE configs' kernels via the library and nvcc-compile them."""
    sys.path.insert(0, ROOT)
    from paper_1907_07875_b200 import gft as G
    import workloads
    os.makedirs(KDIR, exist_ok=True)
    import numpy as np
    todo = {}
    for cfg, dtypes, md in aot_kernel_specs():
        for dt in dtypes:
            plan = G.Plan(cfg.n, cfg.src, cfg.dst, cfg.w, cfg.self_loops, cfg.phi, max_depth=md,
                          dtypes=(dt,))
            for kind in range(4):
                name = plan.kernel_name(kind, dt)
                if name not in todo:
                    todo[name] = plan.kernel_source(kind, dt)
            if md == cfg.max_depth:
                # the fused heat-kernel filter exp(-lambda) timed by bench.py
                filt = G.Filter(plan, np.exp(-plan.eigenvalues()), dtypes=(dt,))
                todo.setdefault(filt.kernel_name(dt), filt.kernel_source(dt))
                if dt == "f32" and cfg.n % 32 == 0:
                    # tensor-core dense comparison kernels timed by bench.py
                    dplan = G.Plan(cfg.n, cfg.src, cfg.dst, cfg.w, cfg.self_loops, cfg.phi, max_depth=md,
                                   dtypes=(dt,), dense_tc=True)
                    for kind in (2, 3):
                        todo.setdefault(dplan.kernel_name(kind, dt), dplan.kernel_source(kind, dt))
    for case in workloads.RIGHT_HAAR_BENCH_CASES:
        # right Haar plans (and their one-block ablation) timed by bench.py
        n, s, d, w, loops, norm = workloads.right_haar_bench_graph(case)
        for rh in (True, False):
            plan = G.Plan(n, s, d, w, loops, dtypes=(case[4],), normalized=norm, right_haar=rh)
            for kind in (0, 1):
                todo.setdefault(plan.kernel_name(kind, case[4]), plan.kernel_source(kind, case[4]))
    for label, variant, kw in workloads.approx_bench_plans():
        # Sec. VI-B comparison (exact / approximate / Haar + approximate) timed by bench.py
        s, d, w = workloads.APPROX_BENCH_GRAPHS[label][0]()
        kw = dict(kw)
        phi = kw.pop("phi")
        plan = G.Plan(64, s, d, w, None, phi, dtypes=("f32",), **kw)
        for kind in ((0, 1, 2) if variant == "haar" else (0, 1)):
            todo.setdefault(plan.kernel_name(kind, "f32"), plan.kernel_source(kind, "f32"))
    s, d, w, loops, _ = workloads.smoke_bipartite32()   # __graft_entry__.smoke()'s tcgen05 case
    plan = G.Plan(64, s, d, w, loops, dtypes=("f32",), normalized=True)
    for kind in (0, 1):
        todo.setdefault(plan.kernel_name(kind, "f32"), plan.kernel_source(kind, "f32"))
    nvcc = os.path.join(CUDA_HOME, "bin", "nvcc")
    pending = [(n, s) for n, s in todo.items() if not os.path.exists(os.path.join(KDIR, n + ".cubin"))]
    with tempfile.TemporaryDirectory() as td:
        procs = []
        for name, src in pending:
            cu = os.path.join(td, name + ".cu")
            with open(cu, "w") as f:
                f.write(src)
            out = os.path.join(KDIR, name + ".cubin")
            cmd = [nvcc, "-cubin", ARCH, "-lineinfo", "-O3", "-std=c++17", "-o", out + ".tmp", cu]
            procs.append((name, out, cmd))
        running = []
        while procs or running:
            while procs and len(running) < jobs:
                name, out, cmd = procs.pop()
                running.append((name, out, cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE,
                                                                 stderr=subprocess.STDOUT)))
            name, out, cmd, p = running.pop(0)
            o = p.communicate()[0].decode()
            if p.returncode != 0:
                raise RuntimeError("nvcc failed for %s:\n%s" % (name, o[-4000:]))
            os.replace(out + ".tmp", out)
    # prune cubins that no longer correspond to a generated kernel
    for f in os.listdir(KDIR):
        if (f.endswith(".cubin") and f[:-6] not in todo) or f.endswith(".cubin.tmp"):
            os.remove(os.path.join(KDIR, f))
    if verbose:
        print("AOT cubins: %d (%d compiled now) in %s" % (len(todo), len(pending), KDIR))
    return sorted(todo)


PEAKS_LIB = os.path.join(LIBDIR, "libgftpeaks.so")


def build_peaks(verbose=True):
    """csrc/peaks.cu -> _lib/libgftpeaks.so: the same-run FFMA / DFMA / tcgen05-TF32 peak
    microbenchmarks bench.py divides by (a measurement tool, not the GFT product path)."""
    src = os.path.join(CSRC, "peaks.cu")
    with open(src, "rb") as f:
        stamp = hashlib.sha256(f.read()).hexdigest()
    sf = PEAKS_LIB + ".stamp"
    if os.path.exists(PEAKS_LIB) and os.path.exists(sf) and open(sf).read() == stamp:
        return PEAKS_LIB
    nvcc = os.path.join(CUDA_HOME, "bin", "nvcc")
    cmd = [nvcc, "-shared", "-Xcompiler", "-fPIC", ARCH, "-lineinfo", "-O3", "-o", PEAKS_LIB + ".tmp", src]
    subprocess.check_call(cmd)
    os.replace(PEAKS_LIB + ".tmp", PEAKS_LIB)
    with open(sf, "w") as f:
        f.write(stamp)
    if verbose:
        print("built", PEAKS_LIB)
    return PEAKS_LIB


def build_c_example(verbose=True):
    """examples/gft_example.c: a plain-C consumer of the C ABI (libgft + CUDA runtime)."""
    exe = os.path.join(LIBDIR, "gft_example")
    cmd = ["gcc", "-O2", "-std=c11", "-Wall", "-I", os.path.join(ROOT, "include"),
           "-I", os.path.join(CUDA_HOME, "include"), os.path.join(ROOT, "examples", "gft_example.c"),
           "-L", LIBDIR, "-lgft", "-L", os.path.join(CUDA_HOME, "lib64"), "-lcudart",
           "-Wl,-rpath,$ORIGIN", "-Wl,-rpath," + os.path.join(CUDA_HOME, "lib64"), "-lm", "-o", exe]
    subprocess.check_call(cmd)
    if verbose:
        print("built", exe)
    return exe


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--no-aot", action="store_true")
    a = ap.parse_args(argv)
    build_library(force=a.force)
    build_c_example()
    build_peaks()
    if not a.no_aot:
        build_aot_cubins()


if __name__ == "__main__":
    main()
