"""Randomised GPU parity sweep over plan shapes (seeded): graph family x size x dtype x plan
options, each through forward and inverse against the oracle.  Catches codegen corner cases
the config tests do not reach (FIX scale ops, odd n with tensor cores off, right stages
inside Haar levels, approximate leaves next to exact ones, n % 4 != 0 bulk layouts)."""
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


def _case(seed):
    rng = np.random.default_rng(1000 + seed)
    kind = ["symmetric", "bipartite_norm", "tree", "random", "rbg"][seed % 5]
    dtype = "f64" if seed % 3 == 0 else "f32"
    n = int(rng.integers(5, 101 if dtype == "f64" else 129))
    kw = {}
    if kind == "symmetric":
        s, d, w, loops, phi = workloads.random_symmetric_graph(rng, n, density=float(rng.uniform(0.1, 0.6)),
                                                               fixed_frac=float(rng.uniform(0, 0.5)))
        L = oracle.laplacian(n, s, d, w, loops)
    elif kind == "bipartite_norm":
        a = int(rng.integers(2, n - 1))
        s, d, w, loops, _ = workloads.random_bipartite_graph(rng, a, n - a, density=0.3)
        phi = None
        kw["normalized"] = True
        L = oracle.normalized_laplacian(oracle.laplacian(n, s, d, w, loops))
    elif kind == "tree":
        parent = [-1] + [int(rng.integers(0, i)) for i in range(1, n)]
        s, d, w = workloads._edges([(p, i) for i, p in enumerate(parent) if p >= 0])
        loops, phi = None, None
        L = oracle.laplacian(n, s, d, w)
    elif kind == "rbg":
        m = max(2, n // 2)
        n = 2 * m
        s, d, w, loops, _ = workloads.regular_bipartite_graph(rng, m, 3, loop=float(rng.uniform(0, 1)))
        phi = None
        L = oracle.laplacian(n, s, d, w, loops)
    else:
        pairs = [(i, j) for i in range(n) for j in range(i + 1, n) if rng.random() < 0.15]
        s, d, w = workloads._edges(pairs, rng.uniform(0.2, 2.0, len(pairs)))
        loops, phi = rng.uniform(0, 0.3, n), None
        L = oracle.laplacian(n, s, d, w, loops)
    if seed % 7 == 4:
        kw["no_tensor_cores"] = True
    if seed % 6 == 5:    # Haar + approximate: the oracle then is the plan's own U_hat check below
        kw["approx_layers"] = int(rng.integers(0, 30))
    return n, (s, d, w, loops, phi), dtype, kw, L


# GFT_FUZZ_SEEDS=a:b widens the sweep (the default suite runs seeds 0..39)
_SEEDS = range(*(int(v) for v in __import__("os").environ.get("GFT_FUZZ_SEEDS", "0:40").split(":")))


@pytest.mark.parametrize("seed", _SEEDS)
def test_random_plan_parity(seed):
    n, (s, d, w, loops, phi), dtype, kw, L = _case(seed)
    plan = G.Plan(n, s, d, w, loops, phi, dtypes=(dtype,), **kw)
    if "approx_layers" in kw:
        # approximate plan: the kernels must apply the plan's U_hat (orthogonal, checked in
        # fp64 here) -- its agreement with the truncated-Jacobi oracle is tested separately
        Uh = plan.basis()
        assert np.abs(Uh.T @ Uh - np.eye(n)).max() < 1e-10
        X = torch.randn(333, n, generator=torch.Generator().manual_seed(seed), dtype=TDT[dtype])
        Y = plan.forward(X.cuda())
        Xr = plan.inverse(Y)
        torch.cuda.synchronize()
        ref = X.numpy().astype(np.float64) @ Uh
        assert oracle.relative_error(Y.cpu().numpy(), ref).max() <= TOL[dtype]
        assert oracle.relative_error(Xr.cpu().numpy(), X.numpy()).max() <= 2 * TOL[dtype]
        return
    lam_o, U_o = oracle.gft_basis(L)
    X = torch.randn(777, n, generator=torch.Generator().manual_seed(seed), dtype=TDT[dtype])
    Y = plan.forward(X.cuda())
    Xr = plan.inverse(Y)
    torch.cuda.synchronize()
    Y_o = oracle.forward(X.numpy(), U_o)
    U_f = plan.basis()
    # (1) the kernels apply exactly the plan's basis: against X U_f in fp64 at the dtype tolerance
    ref_f = X.numpy().astype(np.float64) @ U_f
    assert oracle.relative_error(Y.cpu().numpy(), ref_f).max() <= TOL[dtype], (seed, n, dtype, kw)
    # (2) the plan's basis agrees with the oracle's per eigen-cluster; for random spectra with
    # nearly (not exactly) repeated eigenvalues two correct eigensolves may differ by the
    # Davis-Kahan bound sin(theta) <= |r|_2 / gap (r = residual L u - lambda u of either side;
    # DESIGN.md reading A-5a), so the tolerance is the larger of that bound and the dtype's
    R = oracle.cluster_rotation(U_o, U_f, lam_o)
    gaps = np.diff(lam_o)
    gap = gaps[gaps > 1e-9 * max(1, abs(lam_o).max())].min(initial=1.0)
    res = np.abs(L @ U_o - U_o * lam_o).max() + plan.info()["residual"]
    tol = max(TOL[dtype], np.sqrt(n) * res / gap)
    e = oracle.aligned_error(Y.cpu().numpy(), Y_o, R)
    assert e.max() <= tol, (seed, n, dtype, kw, plan.leaf_sizes(), e.max(), tol)
    assert oracle.relative_error(Xr.cpu().numpy(), X.numpy()).max() <= 2 * TOL[dtype]
