"""C-ABI boundary tests that need no GPU: the library loads, exports every symbol the
header declares, and reports errors as status codes (never aborts)."""
import os
import re

import numpy as np
import pytest

import workloads
from paper_1907_07875_b200 import gft as G

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    with open(os.path.join(ROOT, "include", "gft.h")) as f:
        text = f.read()
    return sorted(set(re.findall(r"^GFT_API\s+[\w\s\*]*?\b(gft_\w+)\s*\(", text, flags=re.M)))


def test_library_exports_every_header_symbol():
    L = G.lib()
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(L, s), s
    assert sorted(G.EXPORTS) == syms
    assert G.gft_abi_version() == 2


def test_library_has_no_hard_cuda_dependency():
    # libcuda / libnvrtc are dlopen-ed so the library loads on CPU-only hosts
    import subprocess
    out = subprocess.run(["ldd", G.LIB_PATH], capture_output=True, text=True).stdout
    assert "libcuda" not in out and "libnvrtc" not in out


def test_status_strings():
    for code, name in G.STATUS.items():
        assert G.gft_status_str(code) == name


def _path(n):
    return workloads.path_graph(n)


@pytest.mark.parametrize("case,status", [
    ("bad_index", "GFT_ERR_INVALID_ARG"),
    ("self_edge", "GFT_ERR_INVALID_ARG"),
    ("duplicate", "GFT_ERR_INVALID_ARG"),
    ("nan", "GFT_ERR_INVALID_ARG"),
    ("inf_loop", "GFT_ERR_INVALID_ARG"),
    ("not_involution", "GFT_ERR_NOT_INVOLUTION"),
    ("phi_range", "GFT_ERR_NOT_INVOLUTION"),
    ("not_symmetric", "GFT_ERR_NOT_SYMMETRIC"),
    ("loop_asym", "GFT_ERR_NOT_SYMMETRIC"),
    ("n0", "GFT_ERR_INVALID_ARG"),
])
def test_plan_create_errors(case, status):
    s, d, w = _path(5)
    loops, phi, n = None, None, 5
    if case == "bad_index":
        d = d.copy(); d[0] = 7
    elif case == "self_edge":
        d = d.copy(); d[1] = s[1]
    elif case == "duplicate":
        s = np.append(s, 1); d = np.append(d, 0); w = np.append(w, 1.0)
    elif case == "nan":
        w = w.copy(); w[2] = np.nan
    elif case == "inf_loop":
        loops = np.zeros(5); loops[1] = np.inf
    elif case == "not_involution":
        phi = np.array([1, 2, 0, 3, 4])
    elif case == "phi_range":
        phi = np.array([4, 3, 2, 1, 9])
    elif case == "not_symmetric":
        w = w.copy(); w[0] = 2.0
        phi = np.array([4, 3, 2, 1, 0])
    elif case == "loop_asym":
        loops = np.zeros(5); loops[0] = 1.0
        phi = np.array([4, 3, 2, 1, 0])
    elif case == "n0":
        n = 0
        s = d = np.zeros(0, np.int32); w = np.zeros(0)
    with pytest.raises(G.GFTError) as ei:
        G.Plan(n, s, d, w, loops, phi, host_only=True)
    assert ei.value.name == status
    assert G.gft_last_error() != ""


def test_zero_weights_dropped_and_negative_accepted():
    s, d, w = _path(4)
    w = np.array([1.0, 0.0, -0.5])
    p = G.Plan(4, s, d, w, host_only=True)
    assert p.info()["residual"] < 1e-12


def test_device_calls_fail_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    s, d, w = _path(8)
    p = G.Plan(8, s, d, w, dtypes=("f32",))
    with pytest.raises(G.GFTError) as ei:
        G.gft_forward(p.handle, 16, 16, 4, G.GFT_F32, 0)
    assert ei.value.name in ("GFT_ERR_NO_DEVICE", "GFT_ERR_COMPILE")
    # batch == 0 is a no-op, NULL pointers are rejected before touching the device
    G.gft_forward(p.handle, 16, 16, 0, G.GFT_F32, 0)
    with pytest.raises(G.GFTError) as ei:
        G.gft_forward(p.handle, 0, 16, 4, G.GFT_F32, 0)
    assert ei.value.name == "GFT_ERR_INVALID_ARG"
    with pytest.raises(G.GFTError) as ei:
        G.gft_forward(p.handle, 17, 16, 4, G.GFT_F32, 0)
    assert ei.value.name == "GFT_ERR_ALIGNMENT"
    with pytest.raises(G.GFTError) as ei:
        G.gft_forward(p.handle, 16, 16, 4, G.GFT_F64, 0)    # f64 not prepared
    assert ei.value.name == "GFT_ERR_UNSUPPORTED"


def test_host_only_plan_has_no_kernels():
    s, d, w = _path(6)
    p = G.Plan(6, s, d, w, host_only=True)
    with pytest.raises(G.GFTError) as ei:
        p.kernel_source(0, "f32")
    assert ei.value.name == "GFT_ERR_UNSUPPORTED"


def test_kernel_source_is_plan_specialised():
    cfg = workloads.config("cfg1")
    p = G.Plan.from_config(cfg)
    src = p.kernel_source(G.K_FAST_FWD, "f32")
    name = p.kernel_name(G.K_FAST_FWD, "f32")
    assert name in src and "gft_body" in src and "cp.async.bulk" in src
    # 7 Haar units -> 7 add/sub pairs (the CUDA-core skeleton keeps FADD pairs), leaves 1,1,2,4
    # -> 22 multiplies (FMA immediates)
    assert src.count("= a_ + b_;") == 7 and src.count("fma.rn.f32x2") == 0
    assert src.count("__fmul_rn(") + src.count("__fmaf_rn(") == 22
    # inverse and dense kernels differ
    assert p.kernel_name(G.K_FAST_INV, "f32") != name
    assert p.kernel_source(G.K_DENSE_FWD, "f32").count("__fmaf_rn(") + \
        p.kernel_source(G.K_DENSE_FWD, "f32").count("__fmul_rn(") == 64


def test_nvrtc_compiles_generated_kernels_on_cpu():
    """Kernel generation + NVRTC compilation need no GPU (module loading does)."""
    cfg = workloads.config("cfg2b")
    p = G.Plan.from_config(cfg, no_cubin_cache=True, dtypes=("f32",))
    p.compile("f32")
    assert p.info()["kernels_ready"] & 1


def test_tuning_record_get_set_on_cpu():
    """gft_plan_tuning_get / _set (no GPU): the record reflects the kernel's geometry, a set
    regenerates the kernel with it (source prelude), survives a save/load round trip when
    re-applied, and invalid or unrealisable records are rejected."""
    cfg = workloads.config("cfg3")
    p = G.Plan.from_config(cfg, dtypes=("f32",))
    rec = p.tuning("f32", kinds=(0, 1))
    assert rec[0] == (4, 2, 3, 150, -1)      # tuning.tsv: fma 25 f32 4 2 3 pace=150 obuf=2
    name0 = p.kernel_name(0, "f32")
    p.set_tuning({0: (2, 2, 8, 150)}, "f32")
    src = p.kernel_source(0, "f32")
    for line in ("#define GFT_R 2", "#define GFT_STAGES 2", "#define GFT_WARPS 8", "#define GFT_PACE_NS 150"):
        assert line in src
    assert p.kernel_name(0, "f32") != name0 and p.tuning("f32", (0,))[0] == (2, 2, 8, 150, -1)
    p.set_tuning({0: (2, 2, 8, 0)}, "f32")
    assert "#define GFT_PACE_NS" not in p.kernel_source(0, "f32")
    # wisdom round trip: plan bytes + record -> identical kernel
    p.set_tuning({0: (1, 3, 8, 300)}, "f32")
    q = G.Plan.load(p.save(), dtypes=("f32",))
    q.set_tuning(p.tuning("f32", (0,)), "f32")
    assert q.kernel_name(0, "f32") == p.kernel_name(0, "f32")
    # the serialised plan carries the non-default records itself (tuning trailer)
    blob = p.save()
    r = G.Plan.load(blob, dtypes=("f32",))
    assert r.kernel_name(0, "f32") == p.kernel_name(0, "f32")
    assert r.kernel_name(1, "f32") == p.kernel_name(1, "f32")          # untouched kind: default
    untuned = G.Plan.from_config(cfg, dtypes=("f32",))
    assert len(untuned.save()) < len(blob)                                # no trailer when untuned
    for bad in (blob + b"x", blob[:-1], blob[:-24] + b"\x00" * 24):
        with pytest.raises(G.GFTError) as ei:
            G.Plan.load(bad, dtypes=("f32",))
        assert ei.value.name == "GFT_ERR_INVALID_ARG"
    for bad in ((3, 2, 4, 0), (1, 1, 4, 0), (1, 2, 0, 0), (1, 2, 4, -1), (8, 8, 16, 0)):
        with pytest.raises(G.GFTError) as ei:
            p.set_tuning({0: bad}, "f32")
        assert ei.value.name == "GFT_ERR_INVALID_ARG"
    for bad in ((2, 2, 8, 0, 1),):                         # FMA kernel with a tc_variant
        with pytest.raises(G.GFTError) as ei:
            p.set_tuning({0: bad}, "f32")
        assert ei.value.name == "GFT_ERR_INVALID_ARG"
    # tensor-core kernels: the record is the tcgen05 variant; it round-trips through the bytes
    t = G.Plan.from_config(workloads.config("cfg5b"), dtypes=("f32",))
    assert t.tuning("f32", (0,))[0] == (-1, -1, -1, -1, 2)          # IO-split warp-specialised (n = 128)
    t.set_tuning({0: (-1, -1, -1, -1, 0)}, "f32")                    # plain CTA pair
    assert "fwdtc2_" in t.kernel_name(0, "f32") and t.tuning("f32", (0,))[0][4] == 0
    t.set_tuning({0: (-1, -1, -1, -1, 3)}, "f32")                    # single CTA
    assert "fwdtc_" in t.kernel_name(0, "f32") and t.tuning("f32", (0,))[0][4] == 3
    u = G.Plan.load(t.save(), dtypes=("f32",))
    assert u.kernel_name(0, "f32") == t.kernel_name(0, "f32")
    for bad in ((1, 2, 4, 0), (-1, -1, -1, -1, 7)):
        with pytest.raises(G.GFTError) as ei:
            t.set_tuning({0: bad}, "f32")
        assert ei.value.name == "GFT_ERR_INVALID_ARG"


def test_tuning_table_kind_and_work_keys():
    """tuning.tsv entries keyed by kind= and work= reach only their kernels (most specific
    match wins): cfg4's fused filter and cfg1's inverse have their own measured geometry."""
    def geo(src):
        return tuple(int(re.search(r"#define %s (\d+)" % k, src).group(1)) for k in ("GFT_R", "GFT_STAGES", "GFT_WARPS"))

    def pace(src):
        m = re.search(r"#define GFT_PACE_NS (\d+)", src)
        return int(m.group(1)) if m else 0

    def obuf(src):
        m = re.search(r"#define GFT_OBUF (\d+)", src)
        return int(m.group(1)) if m else 0

    c4 = G.Plan.from_config(workloads.config("cfg4"), dtypes=("f32",))
    src = c4.kernel_source(0, "f32")
    assert geo(src) == (1, 3, 3) and pace(src) == 150 and obuf(src) == 2
    f4 = G.Filter(c4, np.ones(64), dtypes=("f32",))
    src = f4.kernel_source("f32")
    assert geo(src) == (1, 2, 8) and pace(src) == 150 and obuf(src) == 0
    c5 = G.Plan.from_config(workloads.config("cfg5a"), dtypes=("f32",))
    assert geo(c5.kernel_source(0, "f32")) == (1, 2, 8) and obuf(c5.kernel_source(0, "f32")) == 0
    # cfg5a's inverse shares the forward's geometry (chosen by the sustained regime, r50 / r51)
    assert geo(c5.kernel_source(1, "f32")) == (1, 2, 8) and obuf(c5.kernel_source(1, "f32")) == 0
    c1 = G.Plan.from_config(workloads.config("cfg1"), dtypes=("f32",))
    for k in (0, 1):   # kind=fwd / kind=inv entries (r12)
        src = c1.kernel_source(k, "f32")
        assert geo(src) == (8, 3, 3) and pace(src) == 150 and obuf(src) == 2
    f1 = G.Filter(c1, np.ones(8), dtypes=("f32",))   # kind=filter keeps its own entry
    assert geo(f1.kernel_source("f32")) == (8, 2, 8) and pace(f1.kernel_source("f32")) == 150
    # the dense kernels of cfg1 take the plain n = 8 entry
    assert geo(c1.kernel_source(2, "f32")) == (8, 3, 4) and pace(c1.kernel_source(2, "f32")) == 0


def test_packed_ffma2_units_opt_in(monkeypatch):
    """GFT_FFMA2_UNITS=1 (opt-in) turns the tcgen05 kernels' Haar units into single packed FFMA2
    ops ({b,b}*{1,-1}+{a,a}), one per unit (cfg5b: 64 in the stager); the default and the
    CUDA-core kernels keep FADD pairs."""
    cfg = workloads.config("cfg5b")
    p = G.Plan.from_config(cfg, dtypes=("f32",))
    assert p.kernel_source(0, "f32").count("fma.rn.f32x2") == 0
    monkeypatch.setenv("GFT_FFMA2_UNITS", "1")
    p = G.Plan.from_config(cfg, dtypes=("f32",))
    for k in (0, 1):
        src = p.kernel_source(k, "f32")
        assert "tc3s_" in p.kernel_name(k, "f32")
        assert src.count("fma.rn.f32x2") == p.info()["units_per_level"][0] == 64
        assert "0xBF8000003F800000ull" in src
    c1 = G.Plan.from_config(workloads.config("cfg1"), dtypes=("f32",))
    assert c1.kernel_source(0, "f32").count("fma.rn.f32x2") == 0


def test_binding_validates_output_tensors():
    """The binding passes raw pointers: an output tensor that does not mirror the input (host vs
    device, shape, dtype, strides) must be refused before the library is called."""
    torch = pytest.importorskip("torch")
    p = G.Plan.from_config(workloads.config("cfg1"), dtypes=("f32",), host_only=True)
    a = torch.zeros(16, 8)
    G._check_pair(a, torch.empty_like(a), 8, cuda=False)
    G._check_pair(a, a, 8, cuda=False)                       # in place
    for bad in (torch.zeros(8, 8), torch.zeros(16, 8, dtype=torch.float64), torch.zeros(8, 16).t(),
                torch.zeros(16, 8, dtype=torch.float16), torch.zeros(16 * 8)):
        with pytest.raises(ValueError):
            G._check_pair(a, bad, 8, cuda=False)
    with pytest.raises(ValueError):
        G._check_pair(a, torch.empty_like(a), 8, cuda=True)  # device call with host tensors
    with pytest.raises(ValueError):
        p.forward(a)                                         # host tensor to a device entry point
    ws = torch.zeros(2 * 16 * 8)
    with pytest.raises(ValueError):
        p.execute_host(0, a, torch.zeros(8, 8), ws, 16)      # output smaller than the input
    with pytest.raises(ValueError):
        p.execute_host(0, a, torch.empty_like(a), ws, 16)    # workspace must be a CUDA tensor


def test_binding_validates_host_array_sizes():
    """Array lengths the C side cannot see are checked by the binding."""
    with pytest.raises(ValueError):
        G.gft_laplacian(4, [0, 1], [1, 2], [1.0, 1.0], self_loops=[0.5, 0.5])      # loops shorter than n
    L = G.gft_laplacian(4, [0, 1, 2], [1, 2, 3], [1.0, 1.0, 1.0])
    with pytest.raises(ValueError):
        G.gft_decompose(L, [3, 2, 1])                                             # phi shorter than n
    with pytest.raises(ValueError):
        G.gft_decompose(L[:3], [3, 2, 1, 0])                                      # L not square
    with pytest.raises(ValueError):
        G.gft_find_involution(L[:, :3])
    p = G.Plan.from_config(workloads.config("cfg1"), dtypes=("f32",))
    with pytest.raises(ValueError):
        p.set_tuning({0: (8, 3, 4)}, "f32")                                        # record too short
