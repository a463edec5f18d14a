"""GPU parity: the generated sm_100a kernels (through the C ABI) against the CPU oracle.

Metric (readings A-4, A-17; north star): per-signal relative L2 error after aligning the
plan basis to the oracle basis cluster by cluster (e_b), and the basis-free per-cluster
energy error (e'_b); max over the batch <= 1e-5 (fp32) / 1e-12 (fp64).  Simple
eigenvalues are additionally compared coefficient by coefficient, signed."""
import concurrent.futures as cf
import functools

import numpy as np
import pytest

import oracle
import workloads
from paper_1907_07875_b200 import gft as G

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = {"f32": 1e-5, "f64": 1e-12}
TDT = {"f32": torch.float32, "f64": torch.float64}


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.init()


@functools.lru_cache(maxsize=None)
def oracle_basis(name):
    cfg = workloads.config(name)
    L = oracle.laplacian(cfg.n, cfg.src, cfg.dst, cfg.w, cfg.self_loops)
    return oracle.gft_basis(L)


@functools.lru_cache(maxsize=None)
def plan_for(name, dtype, max_depth=None):
    cfg = workloads.config(name)
    kw = {"dtypes": (dtype,)}
    if max_depth is not None:
        kw["max_depth"] = max_depth
    return G.Plan.from_config(cfg, **kw)


def check_forward(Y_hat, X, lam_o, U_o, U_f, tol):
    Y_o = oracle.forward(X, U_o)
    R = oracle.cluster_rotation(U_o, U_f, lam_o)
    e = oracle.aligned_error(Y_hat, Y_o, R)
    e2 = oracle.energy_error(Y_hat, Y_o, lam_o)
    assert e.max() <= tol, "aligned error %.3e" % e.max()
    assert e2.max() <= tol, "energy error %.3e" % e2.max()
    norms = np.linalg.norm(Y_o, axis=1)
    for C in oracle.clusters(lam_o):
        if len(C) == 1:
            k = C[0]
            d = np.abs(np.asarray(Y_hat, np.float64)[:, k] - Y_o[:, k]) / norms
            assert d.max() <= tol, "coefficient %d error %.3e" % (k, d.max())
    return e.max(), e2.max()


def roundtrip_inputs(name, batch, dtype):
    cfg = workloads.config(name)
    X = workloads.signals(cfg, batch=batch, dtype=dtype)
    return cfg, X


CASES = [("cfg1", "f32", None), ("cfg1", "f32", 1), ("cfg2", "f32", None), ("cfg2b", "f32", None),
         ("cfg3", "f32", None), ("cfg4", "f32", None), ("cfg4", "f64", None), ("cfg5a", "f32", None),
         ("cfg5b", "f32", None)]


@pytest.mark.parametrize("name,dtype,max_depth", CASES)
def test_fast_forward_inverse_vs_oracle(name, dtype, max_depth):
    batch = 4099           # several tiles + a ragged tail for every layout
    cfg, X = roundtrip_inputs(name, batch, dtype)
    plan = plan_for(name, dtype, max_depth)
    lam_o, U_o = oracle_basis(name)
    U_f = plan.basis()
    tol = TOL[dtype]
    Xd = X.cuda()
    Y = plan.forward(Xd)
    torch.cuda.synchronize()
    check_forward(Y.cpu().numpy(), X.numpy(), lam_o, U_o, U_f, tol)
    # inverse of the forward output gives X back
    Xr = plan.inverse(Y)
    torch.cuda.synchronize()
    assert oracle.relative_error(Xr.cpu().numpy(), X.numpy()).max() <= 2 * tol
    # inverse of arbitrary coefficients: U_f c = U_o (R c)
    g = torch.Generator().manual_seed(123)
    Cf = torch.randn(batch, cfg.n, generator=g, dtype=torch.float64).to(TDT[dtype])
    Xc = plan.inverse(Cf.cuda())
    torch.cuda.synchronize()
    R = oracle.cluster_rotation(U_o, U_f, lam_o)
    ref = oracle.inverse(Cf.numpy().astype(np.float64) @ R.T, U_o)
    assert oracle.relative_error(Xc.cpu().numpy(), ref).max() <= tol


@pytest.mark.parametrize("name,dtype", [("cfg1", "f32"), ("cfg3", "f32"), ("cfg4", "f32"),
                                        ("cfg4", "f64"), ("cfg5a", "f32"), ("cfg5b", "f32")])
def test_dense_kernel_vs_oracle(name, dtype):
    batch = 2051
    cfg, X = roundtrip_inputs(name, batch, dtype)
    plan = plan_for(name, dtype)
    lam_o, U_o = oracle_basis(name)
    Y = plan.dense_forward(X.cuda())
    Xr = plan.dense_inverse(Y)
    torch.cuda.synchronize()
    check_forward(Y.cpu().numpy(), X.numpy(), lam_o, U_o, plan.basis(), TOL[dtype])
    assert oracle.relative_error(Xr.cpu().numpy(), X.numpy()).max() <= 2 * TOL[dtype]


@pytest.mark.parametrize("batch", [1, 95, 96, 97, 127, 129, 191, 193, 257])
@pytest.mark.parametrize("name,dtype", [("cfg5a", "f32"), ("cfg5b", "f32"), ("cfg4", "f64")])
def test_dense_gemm_ragged_tiles(name, dtype, batch):
    """Register-tiled dense GEMM (tile rows 96 / 192 / 128): partial first and last tiles."""
    cfg, X = roundtrip_inputs(name, batch, dtype)
    plan = plan_for(name, dtype)
    assert "dgfwd" in plan.kernel_name(G.K_DENSE_FWD, dtype)
    lam_o, U_o = oracle_basis(name)
    Y = plan.dense_forward(X.cuda())
    torch.cuda.synchronize()
    check_forward(Y.cpu().numpy(), X.numpy(), lam_o, U_o, plan.basis(), TOL[dtype])


@pytest.mark.parametrize("name", ["cfg4", "cfg5b"])
def test_dense_tensor_core_kernel_vs_oracle(name):
    """GFT_FLAG_DENSE_TC: dense U^T x as one tcgen05 3xTF32 leaf."""
    cfg = workloads.config(name)
    plan = G.Plan.from_config(cfg, dtypes=("f32",), dense_tc=True)
    assert "dfwdtc" in plan.kernel_name(G.K_DENSE_FWD)
    lam_o, U_o = oracle_basis(name)
    X = workloads.signals(cfg, batch=2051, dtype="f32")
    Y = plan.dense_forward(X.cuda())
    Xr = plan.dense_inverse(Y)
    torch.cuda.synchronize()
    check_forward(Y.cpu().numpy(), X.numpy(), lam_o, U_o, plan.basis(), 1e-5)
    assert oracle.relative_error(Xr.cpu().numpy(), X.numpy()).max() <= 2e-5


@pytest.mark.parametrize("batch", [0, 1, 31, 32, 33, 127, 128, 129, 1000])
@pytest.mark.parametrize("name", ["cfg1", "cfg3", "cfg5a", "cfg5b"])   # packed, bulk (odd n), TMA, tcgen05 pair
def test_small_and_ragged_batches(name, batch):
    plan = plan_for(name, "f32")
    cfg = workloads.config(name)
    lam_o, U_o = oracle_basis(name)
    X = workloads.signals(cfg, batch=max(batch, 1), dtype="f32")[:batch].contiguous()
    Xd = X.cuda()
    # sentinel rows before and after Y (16 rows keep Y 16-byte aligned)
    guard = torch.full((batch + 80, cfg.n), 7.0, device="cuda")
    Yd = guard[16:16 + batch]
    if batch == 0:
        plan.forward(Xd, Yd)
        return
    plan.forward(Xd, Yd)
    torch.cuda.synchronize()
    assert torch.all(guard[16 + batch:] == 7.0), "kernel wrote past the end of Y"
    assert torch.all(guard[:16] == 7.0), "kernel wrote before the start of Y"
    check_forward(Yd.cpu().numpy(), X.numpy(), lam_o, U_o, plan.basis(), 1e-5)
    Zd = guard[16:16 + batch]
    plan.inverse(Yd.clone(), Zd)
    torch.cuda.synchronize()
    assert torch.all(guard[16 + batch:] == 7.0) and torch.all(guard[:16] == 7.0)
    assert oracle.relative_error(Zd.cpu().numpy(), X.numpy()).max() <= 2e-5


@pytest.mark.parametrize("name", ["cfg3", "cfg4", "cfg5b"])
def test_in_place_and_determinism(name):
    plan = plan_for(name, "f32")
    cfg = workloads.config(name)
    X = workloads.signals(cfg, batch=5000, dtype="f32").cuda()
    Y1 = plan.forward(X)
    Y2 = plan.forward(X)
    Z = X.clone()
    plan.forward(Z, Z)                 # in place
    torch.cuda.synchronize()
    assert torch.equal(Y1, Y2)         # bitwise reproducible (no atomics)
    assert torch.equal(Y1, Z)
    plan.inverse(Z, Z)
    torch.cuda.synchronize()
    assert oracle.relative_error(Z.cpu().numpy(), X.cpu().numpy()).max() < 2e-5


def test_alignment_error():
    plan = plan_for("cfg5a", "f32")
    buf = torch.zeros(64 * 10 + 1, device="cuda")
    with pytest.raises(G.GFTError) as e:
        G.gft_forward(plan.handle, buf.data_ptr() + 4, buf.data_ptr(), 10, G.GFT_F32, None)
    assert e.value.name == "GFT_ERR_ALIGNMENT"


def test_random_symmetric_graphs_on_gpu():
    """>= 100 random phi-symmetric graphs (n <= 12) through the full GPU path."""
    rng = np.random.default_rng(77)
    cases = []
    for trial in range(120):
        n = int(rng.integers(1, 13))
        s, d, w, loops, phi = workloads.random_symmetric_graph(
            rng, n, density=float(rng.uniform(0.2, 0.9)), negative=bool(trial % 4 == 0))
        plan = G.Plan(n, s, d, w, loops, phi if trial % 2 else None, dtypes=("f32",))
        cases.append((n, s, d, w, loops, plan))
    with cf.ThreadPoolExecutor(16) as ex:       # NVRTC is thread-safe; ctypes drops the GIL
        list(ex.map(lambda c: c[5].compile("f32", kinds=(0, 1)), cases))
    worst = 0.0
    for n, s, d, w, loops, plan in cases:
        L = oracle.laplacian(n, s, d, w, loops)
        lam_o, U_o = oracle.gft_basis(L)
        X = torch.randn(300, n, generator=torch.Generator().manual_seed(n), dtype=torch.float32)
        Y = plan.forward(X.cuda())
        Xr = plan.inverse(Y)
        torch.cuda.synchronize()
        e, _ = check_forward(Y.cpu().numpy(), X.numpy(), lam_o, U_o, plan.basis(), 1e-5)
        worst = max(worst, e)
        assert oracle.relative_error(Xr.cpu().numpy(), X.numpy()).max() <= 2e-5
    assert worst < 1e-5


def test_tensor_core_single_cta_and_pair_variants_agree(monkeypatch):
    """cfg5b through the three tcgen05 variants that apply at n = 128: the IO-split
    warp-specialised pair kernel (default), the plain CTA-pair kernel (GFT_TC_IOSPLIT=0) and
    the single-CTA kernel (GFT_NO_CTA_PAIR=1) -- against the oracle and each other."""
    cfg = workloads.config("cfg5b")
    ws = G.Plan.from_config(cfg, dtypes=("f32",), no_cubin_cache=True)
    monkeypatch.setenv("GFT_TC_IOSPLIT", "0")
    pair = G.Plan.from_config(cfg, dtypes=("f32",), no_cubin_cache=True)
    monkeypatch.delenv("GFT_TC_IOSPLIT")
    monkeypatch.setenv("GFT_NO_CTA_PAIR", "1")
    single = G.Plan.from_config(cfg, dtypes=("f32",), no_cubin_cache=True)
    monkeypatch.delenv("GFT_NO_CTA_PAIR")
    assert "tc3s_" in ws.kernel_name(G.K_FAST_FWD)
    assert "tc2_" in pair.kernel_name(G.K_FAST_FWD) and "tc_" in single.kernel_name(G.K_FAST_FWD)
    lam_o, U_o = oracle_basis("cfg5b")
    X = workloads.signals(cfg, batch=1000, dtype="f32")   # ragged: 1000 = 3 pair tiles + 232 rows
    Xd = X.cuda()
    for plan in (ws, pair, single):
        Y = plan.forward(Xd)
        Xr = plan.inverse(Y)
        torch.cuda.synchronize()
        check_forward(Y.cpu().numpy(), X.numpy(), lam_o, U_o, plan.basis(), 1e-5)
        assert oracle.relative_error(Xr.cpu().numpy(), X.numpy()).max() <= 2e-5
    ref = single.forward(Xd).cpu().numpy()
    # 3xTF32 variants agree to ~1e-7; the fp16x2 warp-specialised kernel differs by its own
    # (smaller) rounding, each within ~1e-6 of the oracle
    assert oracle.relative_error(pair.forward(Xd).cpu().numpy(), ref).max() < 1e-6
    assert oracle.relative_error(ws.forward(Xd).cpu().numpy(), ref).max() < 3e-6


@pytest.mark.parametrize("inverse_small_leaf", [False, True])
def test_tensor_core_kernel_variants_agree(monkeypatch, inverse_small_leaf):
    """n = 64 plans through all four tcgen05 kernels: warp-specialised stager/drainer pair
    kernel (default, kernel_tc3), two-warpgroup pair kernel (GFT_NO_TC_WS), one-warpgroup pair
    kernel (+GFT_NO_TC_2WG) and single-CTA kernel (GFT_NO_CTA_PAIR) -- against the oracle and
    each other.  The second case has a 24-node CUDA-core leaf beside a 40-node tensor-core
    leaf (stager writes its outputs to SMEM for the drainer)."""
    a, b = (24, 40) if inverse_small_leaf else (32, 32)
    s, d, w, loops, _ = workloads.random_bipartite_graph(np.random.default_rng(a), a, b, density=0.3)
    L = oracle.normalized_laplacian(oracle.laplacian(64, s, d, w, loops))
    lam_o, U_o = oracle.gft_basis(L)
    variants = [("tc3_", {}), ("tc2", {"GFT_NO_TC_WS": "1"}),
                ("tc2_", {"GFT_NO_TC_WS": "1", "GFT_NO_TC_2WG": "1"}), ("tc_", {"GFT_NO_CTA_PAIR": "1"})]
    X = torch.randn(1000, 64, generator=torch.Generator().manual_seed(5))   # 3 pair tiles + ragged
    outs = []
    for tag, env in variants:
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        plan = G.Plan(64, s, d, w, loops, dtypes=("f32",), normalized=True, no_cubin_cache=True)
        for k in env:
            monkeypatch.delenv(k)
        assert tag in plan.kernel_name(G.K_FAST_FWD), (tag, plan.kernel_name(G.K_FAST_FWD))
        Y = plan.forward(X.cuda())
        Xr = plan.inverse(Y)
        torch.cuda.synchronize()
        check_forward(Y.cpu().numpy(), X.numpy(), lam_o, U_o, plan.basis(), 1e-5)
        assert oracle.relative_error(Xr.cpu().numpy(), X.numpy()).max() <= 2e-5
        outs.append(Y.cpu().numpy())
    # the 3xTF32 kernels agree to ~1e-7; the default warp-specialised kernel (fp16x2 split when
    # every leaf is on the tensor core) by its own rounding, each within ~1e-6 of the oracle
    for o in outs[2:]:
        assert oracle.relative_error(o, outs[1]).max() < 1e-6
    assert oracle.relative_error(outs[0], outs[1]).max() < 3e-6


@pytest.mark.parametrize("name", ["cfg3", "cfg4"])
def test_normalized_laplacian_gft(name):
    """GFT of D^{-1/2} L D^{-1/2} through the same fused kernels."""
    cfg = workloads.config(name)
    plan = G.Plan.from_config(cfg, dtypes=("f32",), normalized=True)
    L = oracle.normalized_laplacian(oracle.laplacian(cfg.n, cfg.src, cfg.dst, cfg.w, cfg.self_loops))
    lam_o, U_o = oracle.gft_basis(L)
    X = workloads.signals(cfg, batch=3001, dtype="f32")
    Y = plan.forward(X.cuda())
    Xr = plan.inverse(Y)
    torch.cuda.synchronize()
    check_forward(Y.cpu().numpy(), X.numpy(), lam_o, U_o, plan.basis(), 1e-5)
    assert oracle.relative_error(Xr.cpu().numpy(), X.numpy()).max() <= 2e-5


def _random_big_leaf_graph(rng, n, sym):
    """Random weighted graph whose leaves are large (>= 32) so the tcgen05 path is used;
    sizes chosen to exercise K/N padding (k not a multiple of 16 or 32)."""
    if sym:
        s, d, w, loops, phi = workloads.random_symmetric_graph(rng, n, density=0.3, fixed_frac=0.0)
        return s, d, w, loops, phi
    pairs = [(i, j) for i in range(n) for j in range(i + 1, n) if rng.random() < 0.2]
    s = np.array([p[0] for p in pairs], np.int32)
    d = np.array([p[1] for p in pairs], np.int32)
    w = rng.uniform(0.5, 2.0, len(pairs))
    return s, d, w, rng.uniform(0, 0.5, n), None


@pytest.mark.parametrize("n,sym", [(32, False), (64, False), (80, False), (96, True), (100, True),
                                   (128, True), (160, True)])
def test_tensor_core_leaves_general(n, sym):
    """tcgen05 3xTF32 leaves on random graphs (leaf sizes 32..80 incl. padded K/N), against
    the oracle and against the same plan forced onto CUDA-core FMA."""
    rng = np.random.default_rng(n)
    s, d, w, loops, phi = _random_big_leaf_graph(rng, n, sym)
    plan = G.Plan(n, s, d, w, loops, phi, dtypes=("f32",))
    src = plan.kernel_source(G.K_FAST_FWD, "f32")
    assert "tcgen05.mma" in src, plan.leaf_sizes()
    plan.compile("f32", kinds=(0, 1))          # NVRTC, both directions in parallel
    L = oracle.laplacian(n, s, d, w, loops)
    lam_o, U_o = oracle.gft_basis(L)
    X = torch.randn(3000, n, generator=torch.Generator().manual_seed(1), dtype=torch.float32)
    Y = plan.forward(X.cuda())
    Xr = plan.inverse(Y)
    torch.cuda.synchronize()
    check_forward(Y.cpu().numpy(), X.numpy(), lam_o, U_o, plan.basis(), 1e-5)
    assert oracle.relative_error(Xr.cpu().numpy(), X.numpy()).max() <= 2e-5
    if n > 128:
        return      # (mixed TC + FMA leaves; the all-FMA variant takes minutes to JIT)
    # FMA-only variant of the same plan gives the same coefficients (to fp32 rounding)
    fma = G.Plan(n, s, d, w, loops, phi, dtypes=("f32",), no_tensor_cores=True)
    assert "tcgen05.mma" not in fma.kernel_source(G.K_FAST_FWD, "f32")
    Yf = fma.forward(X.cuda())
    torch.cuda.synchronize()
    assert oracle.relative_error(Y.cpu().numpy(), Yf.cpu().numpy()).max() <= 2e-5


@pytest.mark.parametrize("name,dtype", [("cfg2", "f32"), ("cfg3", "f32"), ("cfg4", "f32"),
                                        ("cfg4", "f64"), ("cfg5a", "f32"), ("cfg5b", "f32")])
def test_full_size_sampled(name, dtype):
    """BASELINE full batch in the launch configuration bench.py times: every row is
    checked for Parseval on the GPU side; 3000 sampled rows (incl. the last) vs oracle."""
    cfg = workloads.config(name)
    plan = plan_for(name, dtype)
    X = workloads.signals(cfg, dtype=dtype)
    Xd = X.cuda()
    Y = plan.forward(Xd)
    torch.cuda.synchronize()
    nx = torch.linalg.vector_norm(Xd.double(), dim=1)
    ny = torch.linalg.vector_norm(Y.double(), dim=1)
    assert float(((ny / nx) - 1).abs().max()) < 10 * TOL[dtype]
    rng = np.random.default_rng(0)
    rows = np.unique(np.concatenate([rng.integers(0, cfg.batch, 3000), [cfg.batch - 1, 0]]))
    lam_o, U_o = oracle_basis(name)
    idx = torch.from_numpy(rows).cuda()
    check_forward(Y[idx].cpu().numpy(), X[rows].numpy(), lam_o, U_o, plan.basis(), TOL[dtype])
    Xr = plan.inverse(Y)
    torch.cuda.synchronize()
    err = (Xr[idx].double() - Xd[idx].double()).norm(dim=1) / Xd[idx].double().norm(dim=1)
    assert float(err.max()) <= 2 * TOL[dtype]


def test_execute_host_end_to_end():
    plan = plan_for("cfg4", "f32")
    cfg = workloads.config("cfg4")
    X = workloads.signals(cfg, batch=10000, dtype="f32").pin_memory()
    Y = torch.empty_like(X).pin_memory()
    ws = torch.empty(2 * 4096 * cfg.n, device="cuda")
    plan.execute_host(0, X, Y, ws, 4096)
    torch.cuda.synchronize()
    ref = plan.forward(X.cuda())
    torch.cuda.synchronize()
    assert torch.equal(Y, ref.cpu())


@pytest.mark.parametrize("name,dtype,slots,chunk,batch", [("cfg3", "f32", 3, 1000, 12345),
                                                           ("cfg4", "f64", 4, 777, 5000),
                                                           ("cfg5b", "f32", 2, 256, 1001)])
def test_execute_host_slots_and_ragged_chunks(name, dtype, slots, chunk, batch):
    """Host-buffer path with 2-4 workspace slots (H2D / kernel / D2H stage streams), chunks that do not divide
    the batch, odd row pitch (cfg3), fp64 and the tensor-core kernel; inverse of the forward
    round-trips; results bit-identical to the device-buffer calls."""
    plan = plan_for(name, dtype)
    cfg = workloads.config(name)
    X = workloads.signals(cfg, batch=batch, dtype=dtype).pin_memory()
    Y = torch.empty_like(X).pin_memory()
    Z = torch.empty_like(X).pin_memory()
    ws = torch.empty(slots * chunk * cfg.n, device="cuda", dtype=TDT[dtype])
    plan.execute_host(0, X, Y, ws, chunk)
    plan.execute_host(1, Y, Z, ws, chunk)
    torch.cuda.synchronize()
    ref = plan.forward(X.cuda())
    torch.cuda.synchronize()
    assert torch.equal(Y, ref.cpu())
    assert oracle.relative_error(Z.numpy(), X.numpy()).max() <= 2 * TOL[dtype]


def test_execute_host_concurrent_threads():
    """Four host threads, each with its own caller stream, workspace and data, call the
    host-buffer path at once (the shared stage streams / events are enqueued under a lock):
    every result equals the device-buffer forward."""
    plan = plan_for("cfg2", "f32")
    n = workloads.config("cfg2").n
    jobs = []
    for t in range(4):
        X = torch.randn(50000 + 999 * t, n, generator=torch.Generator().manual_seed(t)).pin_memory()
        jobs.append((X, torch.empty_like(X).pin_memory(), torch.empty(3 * 4096 * n, device="cuda"),
                     torch.cuda.Stream()))

    def run(job):
        X, Y, ws, st = job
        for _ in range(3):
            plan.execute_host(0, X, Y, ws, 4096, st)
        st.synchronize()

    with cf.ThreadPoolExecutor(4) as ex:
        list(ex.map(run, jobs))
    for X, Y, _, _ in jobs:
        ref = plan.forward(X.cuda())
        torch.cuda.synchronize()
        assert torch.equal(Y, ref.cpu())


@pytest.mark.parametrize("kind,n,dtype", [("complete", 64, "f32"), ("complete", 64, "f64"),
                                          ("star", 33, "f32"), ("star", 100, "f64")])
def test_two_sparse_eigenvector_graphs_on_gpu(kind, n, dtype):
    """Lemma 4 graphs: K_64 plans to a pure Haar network (63 units, all
    leaves 1x1); the star keeps one small leaf.  Parity vs the oracle (degenerate spectra:
    aligned per cluster)."""
    if kind == "complete":
        pairs = [(i, j) for i in range(n) for j in range(i + 1, n)]
    else:
        pairs = [(0, i) for i in range(1, n)]
    s = np.array([p[0] for p in pairs], np.int32)
    d = np.array([p[1] for p in pairs], np.int32)
    w = np.ones(len(pairs))
    plan = G.Plan(n, s, d, w, dtypes=(dtype,))
    if kind == "complete":
        assert plan.info()["n_units"] == n - 1 and max(plan.leaf_sizes()) == 1
    L = oracle.laplacian(n, s, d, w)
    lam_o, U_o = oracle.gft_basis(L)
    X = torch.randn(2053, n, generator=torch.Generator().manual_seed(n), dtype=TDT[dtype])
    Y = plan.forward(X.cuda())
    Xr = plan.inverse(Y)
    torch.cuda.synchronize()
    check_forward(Y.cpu().numpy(), X.numpy(), lam_o, U_o, plan.basis(), TOL[dtype])
    assert oracle.relative_error(Xr.cpu().numpy(), X.numpy()).max() <= 2 * TOL[dtype]


@pytest.mark.parametrize("batch", [1, 255, 257, 1000, 70001])
def test_tensor_core_io_split_kernel(batch):
    """The IO-split warp-specialised kernel (default for n > 64 with every leaf on the tensor
    core: two input buffers, box-granular output ring, per-chunk A release, load pacing):
    cfg5b forward / inverse vs the oracle over one, several and a ragged number of pair tiles."""
    cfg = workloads.config("cfg5b")
    plan = G.Plan.from_config(cfg, dtypes=("f32",))
    assert "tc3s_" in plan.kernel_name(G.K_FAST_FWD) and "tc3s_" in plan.kernel_name(G.K_FAST_INV)
    src = plan.kernel_source(G.K_FAST_FWD, "f32")
    assert "#define GFT_IO_SPLIT 1" in src and "#define GFT_LOAD_PACE_NS" in src and "#define GFT_NCH 4" in src
    assert "#define GFT_F16X2 1" in src
    lam_o, U_o = oracle_basis("cfg5b")
    X = workloads.signals(cfg, batch=batch, dtype="f32")
    Y = plan.forward(X.cuda())
    Xr = plan.inverse(Y)
    torch.cuda.synchronize()
    check_forward(Y.cpu().numpy(), X.numpy(), lam_o, U_o, plan.basis(), 1e-5)
    assert oracle.relative_error(Xr.cpu().numpy(), X.numpy()).max() <= 2e-5


def test_tensor_core_plain_pair_ablation(monkeypatch):
    """GFT_TC_IOSPLIT=0 keeps the plain CTA-pair kernel for cfg5b; it stays correct."""
    cfg = workloads.config("cfg5b")
    monkeypatch.setenv("GFT_TC_IOSPLIT", "0")
    plan = G.Plan.from_config(cfg, dtypes=("f32",), no_cubin_cache=True)
    monkeypatch.delenv("GFT_TC_IOSPLIT")
    assert "tc2_" in plan.kernel_name(G.K_FAST_FWD)
    lam_o, U_o = oracle_basis("cfg5b")
    X = workloads.signals(cfg, batch=1000, dtype="f32")
    Y = plan.forward(X.cuda())
    Xr = plan.inverse(Y)
    torch.cuda.synchronize()
    check_forward(Y.cpu().numpy(), X.numpy(), lam_o, U_o, plan.basis(), 1e-5)
    assert oracle.relative_error(Xr.cpu().numpy(), X.numpy()).max() <= 2e-5


@pytest.mark.parametrize("leaves", [1, 2])
def test_tensor_core_ws_chunked_staging(leaves):
    """The in-place warp-specialised kernel (n <= 64) stages and releases A per 32-column
    chunk: a 64-node graph with one 64-leaf (no symmetry: random weights) or a mirror-symmetric
    one with two 32-leaves, forward / inverse vs the oracle over several tiles + a ragged tail."""
    rng = np.random.default_rng(7 + leaves)
    n = 64
    if leaves == 1:
        pairs = [(i, j) for i in range(n) for j in range(i + 1, n) if rng.random() < 0.15]
        w = rng.uniform(0.5, 2.0, len(pairs))
    else:
        half = [(i, j) for i in range(32) for j in range(i + 1, 32) if rng.random() < 0.2]
        wh = rng.uniform(0.5, 2.0, len(half))
        pairs = half + [(63 - i, 63 - j) for i, j in half] + [(i, 63 - i) for i in range(32)]
        w = np.concatenate([wh, wh, np.full(32, 0.7)])
    s = np.array([p[0] for p in pairs], np.int32)
    d = np.array([p[1] for p in pairs], np.int32)
    plan = G.Plan(n, s, d, w, dtypes=("f32",))
    src = plan.kernel_source(G.K_FAST_FWD, "f32")
    assert "tc3_" in plan.kernel_name(G.K_FAST_FWD) and "#define GFT_NCH 2" in src
    assert plan.leaf_sizes() == ([64] if leaves == 1 else [32, 32])
    lam_o, U_o = oracle.gft_basis(oracle.laplacian(n, s, d, w))
    X = torch.randn(5000, n, generator=torch.Generator().manual_seed(leaves))
    Y = plan.forward(X.cuda())
    Xr = plan.inverse(Y)
    torch.cuda.synchronize()
    check_forward(Y.cpu().numpy(), X.numpy(), lam_o, U_o, plan.basis(), 1e-5)
    assert oracle.relative_error(Xr.cpu().numpy(), X.numpy()).max() <= 2e-5


@pytest.mark.parametrize("case", ["wide_f64_leaf", "forced_cfg4_f64"])
def test_streamed_leaf_outputs(monkeypatch, case):
    """Wide rows write leaf outputs straight to SMEM (no y register row): a 96-node f64 leaf
    (automatic), and cfg4 f64 with GFT_STREAM=1 (inverse: outputs reloaded for the reverse
    butterflies) -- both against the oracle, with a ragged batch."""
    if case == "wide_f64_leaf":
        rng = np.random.default_rng(3)
        n = 96
        pairs = [(i, j) for i in range(n) for j in range(i + 1, n) if rng.random() < 0.1]
        s = np.array([p[0] for p in pairs], np.int32)
        d = np.array([p[1] for p in pairs], np.int32)
        w = rng.uniform(0.5, 2.0, len(pairs))
        plan = G.Plan(n, s, d, w, dtypes=("f64",))
        L = oracle.laplacian(n, s, d, w)
        lam_o, U_o = oracle.gft_basis(L)
    else:
        cfg = workloads.config("cfg4")
        monkeypatch.setenv("GFT_STREAM", "1")
        plan = G.Plan.from_config(cfg, dtypes=("f64",), no_cubin_cache=True)
        monkeypatch.delenv("GFT_STREAM")
        n = cfg.n
        lam_o, U_o = oracle_basis("cfg4")
    assert "GFT_STREAM" in plan.kernel_source(G.K_FAST_FWD, "f64")
    X = torch.randn(1001, n, generator=torch.Generator().manual_seed(2), dtype=torch.float64)
    Y = plan.forward(X.cuda())
    Xr = plan.inverse(Y)
    torch.cuda.synchronize()
    check_forward(Y.cpu().numpy(), X.numpy(), lam_o, U_o, plan.basis(), 1e-12)
    assert oracle.relative_error(Xr.cpu().numpy(), X.numpy()).max() <= 2e-12


@pytest.mark.parametrize("case", ["n1", "n2", "edgeless5", "loops_only4", "negative6", "n256_host_only"])
def test_degenerate_graphs(case):
    """Degenerate inputs through the C ABI: 1- and 2-node graphs, no edges (L = 0: the GFT is
    the identity up to order), self-loops only (L diagonal), negative weights (L not PSD), and
    n = 256 planned host-only (the largest n with kernels is 256)."""
    if case == "n256_host_only":
        s, d, w = workloads.cycle_graph(256)
        plan = G.Plan(256, s, d, w, host_only=True)
        assert plan.info()["units_per_level"][0] == 128
        lam = plan.eigenvalues()
        assert np.abs(np.sort(lam) - np.sort(2 - 2 * np.cos(2 * np.pi * np.arange(256) / 256))).max() < 1e-10
        return
    e = np.zeros(0, np.int32)
    if case == "n1":
        n, s, d, w, loops = 1, e, e, np.zeros(0), np.array([0.7])
    elif case == "n2":
        n, s, d, w, loops = 2, np.array([0], np.int32), np.array([1], np.int32), np.array([1.5]), None
    elif case == "edgeless5":
        n, s, d, w, loops = 5, e, e, np.zeros(0), None
    elif case == "loops_only4":
        n, s, d, w, loops = 4, e, e, np.zeros(0), np.array([0.5, 2.0, 1.0, 3.0])
    else:
        n = 6
        s, d, w = workloads._edges([(0, 1), (1, 2), (2, 3), (3, 4), (4, 5), (0, 5), (1, 4)],
                                   [1.0, -0.5, 2.0, -0.5, 1.0, 0.7, -1.2])
        loops = None
    for dtype in ("f32", "f64"):
        plan = G.Plan(n, s, d, w, loops, dtypes=(dtype,))
        L = oracle.laplacian(n, s, d, w, loops)
        lam_o, U_o = oracle.gft_basis(L)
        X = torch.randn(65, n, generator=torch.Generator().manual_seed(n), dtype=TDT[dtype])
        Y = plan.forward(X.cuda())
        Xr = plan.inverse(Y)
        torch.cuda.synchronize()
        check_forward(Y.cpu().numpy(), X.numpy(), lam_o, U_o, plan.basis(), TOL[dtype])
        assert oracle.relative_error(Xr.cpu().numpy(), X.numpy()).max() <= 2 * TOL[dtype]


@pytest.mark.parametrize("n,dtype,force", [(8, "f32", False), (4, "f32", False), (4, "f64", False),
                                           (8, "f64", True), (16, "f32", True)])
@pytest.mark.parametrize("batch", [1, 3, 4, 130, 1001, 70001])
def test_packed_view_mode(monkeypatch, n, dtype, force, batch):
    """Rows of 16/32/64 bytes move as a packed [batch/g, g*n] TMA view with 128-byte box rows
    and 128B swizzle (default for rows <= 32 B, GFT_PACK=1 forces 64-B rows): a cycle plan vs
    the oracle with ragged batches (batch % g signals take the direct path, batch < g too)."""
    s = np.arange(n, dtype=np.int32)
    d = ((s + 1) % n).astype(np.int32)
    w = np.random.default_rng(n).uniform(0.5, 2.0, n)
    if force:
        monkeypatch.setenv("GFT_PACK", "1")
    plan = G.Plan(n, s, d, w, dtypes=(dtype,), no_cubin_cache=force)
    monkeypatch.delenv("GFT_PACK", raising=False)
    src = plan.kernel_source(G.K_FAST_FWD, dtype)
    assert "#define GFT_MODE 2" in src and f"#define GFT_PACK {128 // (n * (8 if dtype == 'f64' else 4))}" in src
    lam_o, U_o = oracle.gft_basis(oracle.laplacian(n, s, d, w))
    X = torch.randn(batch, n, generator=torch.Generator().manual_seed(batch), dtype=TDT[dtype])
    Y = plan.forward(X.cuda())
    Xr = plan.inverse(Y)
    torch.cuda.synchronize()
    check_forward(Y.cpu().numpy(), X.numpy(), lam_o, U_o, plan.basis(), TOL[dtype])
    assert oracle.relative_error(Xr.cpu().numpy(), X.numpy()).max() <= 2 * TOL[dtype]


@pytest.mark.parametrize("which", ["ws_tc3", "f64"])
@pytest.mark.parametrize("batch", [1, 129, 1000])
def test_guard_regions_ws_and_f64(which, batch):
    """Sentinel rows around Y for the warp-specialised tcgen05 kernel (right-Haar 32|32,
    n = 64) and the fp64 FMA kernel (cfg4): nothing written outside Y, Y = X U_f."""
    if which == "ws_tc3":
        n, s_, d_, w_, loops, norm = workloads.right_haar_bench_graph(workloads.RIGHT_HAAR_BENCH_CASES[0])
        plan = G.Plan(n, s_, d_, w_, loops, dtypes=("f32",), normalized=norm)
        assert "tc3" in plan.kernel_name(0, "f32")
        tdt, tol, dt = torch.float32, 1e-5, "f32"
    else:
        cfg = workloads.config("cfg4")
        n = cfg.n
        plan = G.Plan.from_config(cfg, dtypes=("f64",))
        tdt, tol, dt = torch.float64, 1e-12, "f64"
    X = torch.randn(batch, n, generator=torch.Generator().manual_seed(batch), dtype=tdt)
    guard = torch.full((batch + 80, n), 7.0, device="cuda", dtype=tdt)
    Yd = guard[16:16 + batch]
    plan.forward(X.cuda(), Yd)
    torch.cuda.synchronize()
    assert torch.all(guard[:16] == 7.0) and torch.all(guard[16 + batch:] == 7.0)
    ref = X.double().numpy() @ plan.basis()
    err = np.linalg.norm(Yd.cpu().double().numpy() - ref, axis=1) / np.linalg.norm(ref, axis=1)
    assert err.max() <= tol
    plan.close()


@pytest.mark.parametrize("name,dtype,obuf", [("cfg3", "f32", 1), ("cfg3", "f32", 2), ("cfg4", "f64", 1),
                                             ("cfg4", "f32", 2), ("cfg1", "f32", 2)])
@pytest.mark.parametrize("batch", [1, 250, 4099])
def test_fma_io_split_outputs(monkeypatch, name, dtype, obuf, batch):
    """CUDA-core kernel with separate output tiles (IO split, GFT_FMA_OBUF / tuning.tsv obuf=):
    bulk (odd pitch, direct ragged tail), TMA and packed-view modes, forward / inverse /
    fused filter against the oracle on ragged batches."""
    cfg = workloads.config(name)
    monkeypatch.setenv("GFT_FMA_OBUF", str(obuf))
    plan = G.Plan.from_config(cfg, dtypes=(dtype,), no_cubin_cache=True)
    filt = G.Filter(plan, np.exp(-plan.eigenvalues()), dtypes=(dtype,), no_cubin_cache=True)
    monkeypatch.delenv("GFT_FMA_OBUF")
    assert "#define GFT_OBUF %d" % obuf in plan.kernel_source(G.K_FAST_FWD, dtype)
    lam_o, U_o = oracle_basis(name)
    X = workloads.signals(cfg, batch=batch, dtype=dtype)
    Xd = X.cuda()
    Y = plan.forward(Xd)
    Xr = plan.inverse(Y)
    Z = filt.apply(Xd)
    torch.cuda.synchronize()
    check_forward(Y.cpu().numpy(), X.numpy(), lam_o, U_o, plan.basis(), TOL[dtype])
    assert oracle.relative_error(Xr.cpu().numpy(), X.numpy()).max() <= 2 * TOL[dtype]
    Zo = oracle.graph_filter(X.numpy().astype(np.float64), U_o, np.exp(-lam_o))
    assert oracle.relative_error(Z.cpu().numpy(), Zo).max() <= 4 * TOL[dtype]


@pytest.mark.parametrize("name", ["cfg5b", "rh0"])
def test_tensor_core_f16x2_extreme_magnitudes(name):
    """The fp16x2 split of the warp-specialised kernels scales every row by a power of two
    (its largest tensor-core input into [1, 2)) before splitting into fp16 parts: rows spanning
    the fp32 range (1e-30 .. 1e30), rows with one huge and many tiny elements, all-zero rows and
    mixed signs all stay within the per-signal 1e-5 bound, forward and round trip, against the
    oracle (fp64)."""
    if name == "cfg5b":
        cfg = workloads.config("cfg5b")
        plan = G.Plan.from_config(cfg, dtypes=("f32",))
        n = cfg.n
        L = oracle.laplacian(n, cfg.src, cfg.dst, cfg.w, cfg.self_loops)
    else:
        n, s_, d_, w_, loops, norm = workloads.right_haar_bench_graph(workloads.RIGHT_HAAR_BENCH_CASES[0])
        plan = G.Plan(n, s_, d_, w_, loops, dtypes=("f32",), normalized=norm)
        L = oracle.laplacian(n, s_, d_, w_, loops)
        if norm:
            L = oracle.normalized_laplacian(L)
    assert "#define GFT_F16X2 1" in plan.kernel_source(G.K_FAST_FWD, "f32")
    lam_o, U_o = oracle.gft_basis(L)
    g = torch.Generator().manual_seed(11)
    base = torch.randn(64, n, generator=g)
    rows = [base[i] * (10.0 ** e) for i, e in enumerate([-30, -20, -10, -5, 0, 5, 10, 20, 30])]
    spike = torch.randn(n, generator=g) * 1e-6
    spike[3] = 1e4
    rows += [spike, -spike, base[20] * torch.logspace(-8, 8, n), torch.zeros(n)]
    rows += [base[30 + i] for i in range(10)]
    X = torch.stack(rows).float()
    X = torch.cat([X, torch.randn(1000, n, generator=g)])   # + full pair tiles and a ragged tail
    Y = plan.forward(X.cuda())
    Xr = plan.inverse(Y)
    torch.cuda.synchronize()
    Yh, Xn = Y.cpu().numpy().astype(np.float64), X.numpy().astype(np.float64)
    nz = np.abs(Xn).sum(axis=1) > 0
    assert np.all(Yh[~nz] == 0)                                # zero rows stay exactly zero
    check_forward(Yh[nz], Xn[nz], lam_o, U_o, plan.basis(), 1e-5)
    assert oracle.relative_error(Xr.cpu().numpy()[nz], Xn[nz]).max() <= 2e-5


def test_max_size_n256():
    """The largest n with kernels (256): the 256-cycle plan (leaves up to 64, too big for the
    tensor-core tiles at this row width, so the CUDA-core skeleton in stream mode) forward and
    inverse on a ragged batch against the oracle, per eigen-cluster (the cycle's eigenvalues are
    2-fold); the spectrum is also pinned to the closed form 2 - 2 cos(2 pi k / 256)."""
    n = 256
    s, d, w = workloads.cycle_graph(n)
    plan = G.Plan(n, s, d, w, dtypes=("f32",))
    assert "GFT_STREAM" in plan.kernel_source(G.K_FAST_FWD, "f32")
    L = oracle.laplacian(n, s, d, w)
    lam_o, U_o = oracle.gft_basis(L)
    assert np.abs(lam_o - np.sort(2 - 2 * np.cos(2 * np.pi * np.arange(n) / n))).max() < 1e-10
    X = torch.randn(1001, n, generator=torch.Generator().manual_seed(256), dtype=torch.float32)
    Y = plan.forward(X.cuda())
    Xr = plan.inverse(Y)
    torch.cuda.synchronize()
    check_forward(Y.cpu().numpy(), X.numpy(), lam_o, U_o, plan.basis(), TOL["f32"])
    assert oracle.relative_error(Xr.cpu().numpy(), X.numpy()).max() <= 2 * TOL["f32"]
