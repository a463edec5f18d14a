"""GPU parity of plans with right Haar stages (NEXT-2): leaves E | F then
coefficient butterflies (forward) / their transpose before the leaves (inverse), on the
CUDA-core FMA path and on the tcgen05 path (leaves >= 32), plus the fused filter, whose
E | F pair is one block.  Reference: the oracle's eigenbasis of the same Laplacian."""
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


def _graph(kind, a, b, seed):
    rng = np.random.default_rng(seed)
    if kind == "norm":
        s, d, w, loops, _ = workloads.random_bipartite_graph(rng, a, b, density=0.3)
        n = a + b
        L = oracle.normalized_laplacian(oracle.laplacian(n, s, d, w, loops))
        return n, (s, d, w, loops), True, L
    s, d, w, loops, _ = workloads.regular_bipartite_graph(rng, a, 3, loop=0.5)
    n = 2 * a
    return n, (s, d, w, loops), False, oracle.laplacian(n, s, d, w, loops)


def _check(Y_hat, X, lam_o, U_o, U_f, tol):
    Y_o = oracle.forward(X, U_o)
    R = oracle.cluster_rotation(U_o, U_f, lam_o)
    e = oracle.aligned_error(Y_hat, Y_o, R)
    e2 = oracle.energy_error(Y_hat, Y_o, lam_o)
    assert e.max() <= tol, "aligned error %.3e" % e.max()
    assert e2.max() <= tol, "energy error %.3e" % e2.max()
    norms = np.linalg.norm(Y_o, axis=1)
    for C in oracle.clusters(lam_o):
        if len(C) == 1:
            d = np.abs(np.asarray(Y_hat, np.float64)[:, C[0]] - Y_o[:, C[0]]) / norms
            assert d.max() <= tol, "coefficient %d error %.3e" % (C[0], d.max())


CASES = [("norm", 16, 16, "f32"), ("norm", 16, 16, "f64"), ("norm", 13, 20, "f32"),
         ("norm", 5, 9, "f64"), ("reg", 24, 0, "f32"), ("reg", 24, 0, "f64"),
         ("norm", 32, 32, "f32"), ("norm", 40, 56, "f32"), ("reg", 64, 0, "f32"),
         ("norm", 40, 40, "f32"), ("norm", 36, 48, "f32")]


@pytest.mark.parametrize("kind,a,b,dtype", CASES)
def test_right_stage_forward_inverse(kind, a, b, dtype):
    n, (s, d, w, loops), norm, L = _graph(kind, a, b, 17 * a + b)
    plan = G.Plan(n, s, d, w, loops, dtypes=(dtype,), normalized=norm)
    info = plan.info()
    assert info["n_right_stages"] >= 1 and info["n_right_pairs"] >= 1
    src = plan.kernel_source(G.K_FAST_FWD, dtype)
    assert "right Haar stage" in src
    if dtype == "f32" and min(plan.leaf_sizes()) >= 32:
        assert "tcgen05.mma" in src, plan.leaf_sizes()
    lam_o, U_o = oracle.gft_basis(L)
    batch = 4099                                  # several tiles + a ragged tail
    X = torch.randn(batch, n, generator=torch.Generator().manual_seed(n), dtype=TDT[dtype])
    Y = plan.forward(X.cuda())
    Xr = plan.inverse(Y)
    torch.cuda.synchronize()
    tol = TOL[dtype]
    _check(Y.cpu().numpy(), X.numpy(), lam_o, U_o, plan.basis(), tol)
    # forward verified above, so the round trip pins the inverse (pre-units + leaves^T)
    assert oracle.relative_error(Xr.cpu().numpy(), X.numpy()).max() <= 2 * tol


@pytest.mark.parametrize("kind,a,b,dtype", [("norm", 16, 16, "f32"), ("norm", 13, 20, "f64"),
                                            ("norm", 32, 32, "f32")])
def test_right_stage_filter(kind, a, b, dtype):
    n, (s, d, w, loops), norm, L = _graph(kind, a, b, 5 * a + b)
    plan = G.Plan(n, s, d, w, loops, dtypes=(dtype,), normalized=norm)
    assert plan.info()["n_right_stages"] >= 1
    lam = plan.eigenvalues()
    lam_o, U_o = oracle.gft_basis(L)
    X = torch.randn(3001, n, generator=torch.Generator().manual_seed(3), dtype=TDT[dtype])
    tol = TOL[dtype]
    Xn = X.numpy().astype(np.float64)
    # h = lambda -> x L  (no eigensolve on the reference side)
    Y = G.Filter(plan, lam, dtypes=(dtype,)).apply(X.cuda())
    torch.cuda.synchronize()
    err = np.linalg.norm(Y.cpu().numpy() - Xn @ L, axis=1) / (np.linalg.norm(Xn, axis=1) * np.abs(lam).max())
    assert err.max() <= 2 * tol, err.max()
    # heat kernel vs the oracle
    Yh = G.Filter(plan, np.exp(-0.7 * lam), dtypes=(dtype,)).apply(X.cuda())
    torch.cuda.synchronize()
    ref = oracle.graph_filter(X.numpy(), U_o, np.exp(-0.7 * lam_o))
    assert (np.linalg.norm(Yh.cpu().numpy() - ref, axis=1) / np.linalg.norm(Xn, axis=1)).max() <= 2 * tol
    # arbitrary per-coefficient response (splits the pairs) vs two-pass on the same plan
    h = np.random.default_rng(9).uniform(-1, 1, n)
    Yf = G.Filter(plan, h, dtypes=(dtype,)).apply(X.cuda())
    Y2 = plan.inverse(plan.forward(X.cuda()) * torch.from_numpy(h).to(TDT[dtype]).cuda())
    torch.cuda.synchronize()
    assert oracle.relative_error(Yf.cpu().numpy(), Y2.cpu().numpy()).max() <= 4 * tol


@pytest.mark.parametrize("batch", [1, 255, 256, 70001])
def test_split_store_bit_identical(batch, monkeypatch):
    """The in-place warp-specialised tcgen05 kernel's split storer (default) only reorders
    stores and loads: outputs are bit-identical to the single producer / storer thread
    (GFT_TC_SPLIT_STORE=0), for ragged batches of 1 .. several tiles, forward and inverse."""
    n, (s, d, w, loops), norm, _ = _graph("norm", 32, 32, 11)
    X = torch.randn(batch, n, generator=torch.Generator().manual_seed(batch), dtype=torch.float32).cuda()
    outs = []
    for v in ("1", "0"):
        monkeypatch.setenv("GFT_TC_SPLIT_STORE", v)
        p = G.Plan(n, s, d, w, loops, dtypes=("f32",), normalized=norm, no_cubin_cache=True)
        assert "tc3_" in p.kernel_name(0, "f32")
        outs.append((p.forward(X), p.inverse(X), p.kernel_name(0, "f32")))
        p.close()
    torch.cuda.synchronize()
    assert outs[0][2] != outs[1][2]   # two different kernels
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])


@pytest.mark.parametrize("knob", ["GFT_TC_A2=0", "GFT_FFMA2_UNITS=1"])
def test_tc_variants_bit_identical(knob, monkeypatch):
    """Variants that only change scheduling or the instruction form give bit-identical outputs:
    one vs two A buffers in TMEM (GFT_TC_A2) and packed-FFMA2 vs FADD Haar units
    (GFT_FFMA2_UNITS: fma(b, +-1, a) is the exactly rounded a +- b), on a 64|64 right-Haar plan
    (IO-split kernel; coefficient butterflies of both signs after / before the leaves) with a
    ragged batch, forward and inverse."""
    n, (s, d, w, loops), norm, _ = _graph("norm", 64, 64, 5)
    X = torch.randn(70001, n, generator=torch.Generator().manual_seed(3), dtype=torch.float32).cuda()
    outs = []
    for env in ({}, dict([knob.split("=")])):
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        p = G.Plan(n, s, d, w, loops, dtypes=("f32",), normalized=norm, no_cubin_cache=True)
        assert "tc3s_" in p.kernel_name(0, "f32") and p.info()["n_right_pairs"] == 64
        outs.append((p.forward(X), p.inverse(X), p.kernel_name(0, "f32")))
        p.close()
        for k in env:
            monkeypatch.delenv(k)
    torch.cuda.synchronize()
    assert outs[0][2] != outs[1][2]
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])
