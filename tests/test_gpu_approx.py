"""GPU parity of approximate plans (NEXT-4): the generated kernels apply
J Givens layers (+ Haar units) in registers; the reference is the approximate ORACLE's
U_hat (truncated Jacobi, reading R-4) applied in fp64, compared per cluster of approximate
eigenvalues (aligned error, as for the exact GFT) -- plus the round trip."""
import numpy as np
import pytest

import oracle
import workloads
from paper_1907_07875_b200 import gft as G

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = {"f32": 1e-5, "f64": 1e-12}
TDT = {"f32": torch.float32, "f64": torch.float64}
PHI = {"bidiag": np.array([8 * (i % 8) + i // 8 for i in range(64)], np.int32),
       "z": np.array([63 - i for i in range(64)], np.int32)}


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.init()


@pytest.mark.parametrize("name,J,depth,dtype", [("bidiag", 20, 0, "f32"), ("bidiag", 40, 0, "f64"),
                                                ("z", 10, 1, "f32"), ("z", 30, 1, "f64"),
                                                ("bidiag", 5, 1, "f32"), ("z", 0, 0, "f32")])
def test_approximate_plan_kernels_vs_oracle(name, J, depth, dtype):
    s, d, w = workloads.bidiag_grid() if name == "bidiag" else workloads.z_grid()
    L = oracle.laplacian(64, s, d, w)
    phi = PHI[name] if depth else None
    plan = G.Plan(64, s, d, w, None, phi, dtypes=(dtype,), max_depth=depth, approx_layers=J)
    src = plan.kernel_source(G.K_FAST_FWD, dtype)
    assert "approximate" in src and "tcgen05" not in src
    if depth == 0:
        _, _, U_o, lam_o = oracle.truncated_jacobi(L, J)
    else:
        lam_o, U_o = oracle.haar_approx_basis(L, phi, J)
    X = torch.randn(4099, 64, generator=torch.Generator().manual_seed(J), dtype=TDT[dtype])
    Y = plan.forward(X.cuda())
    Xr = plan.inverse(Y)
    torch.cuda.synchronize()
    Y_o = oracle.forward(X.numpy(), U_o)
    R = oracle.cluster_rotation(U_o, plan.basis(), lam_o)   # +-1 per column (signs free)
    tol = TOL[dtype]
    e = oracle.aligned_error(Y.cpu().numpy(), Y_o, R)
    assert e.max() <= tol, e.max()
    assert oracle.relative_error(Xr.cpu().numpy(), X.numpy()).max() <= 2 * tol


def test_approximate_filter_is_dense_block():
    """The fused filter on an approximate plan: U_hat diag(h) U_hat^T, with h = lam_hat
    giving U_hat diag(lam_hat) U_hat^T (the approximation of L the plan represents)."""
    s, d, w = workloads.z_grid()
    plan = G.Plan(64, s, d, w, None, PHI["z"], dtypes=("f32",), max_depth=1, approx_layers=10)
    lam_o, U_o = oracle.haar_approx_basis(oracle.laplacian(64, s, d, w), PHI["z"], 10)
    h = np.exp(-0.3 * plan.eigenvalues())
    X = torch.randn(3001, 64, generator=torch.Generator().manual_seed(2))
    Y = G.Filter(plan, h, dtypes=("f32",)).apply(X.cuda())
    torch.cuda.synchronize()
    ref = oracle.graph_filter(X.numpy(), U_o, np.exp(-0.3 * lam_o))
    err = np.linalg.norm(Y.cpu().numpy() - ref, axis=1) / np.linalg.norm(X.numpy().astype(np.float64), axis=1)
    assert err.max() <= 2e-5, err.max()


@pytest.mark.parametrize("name,J,depth,force", [("bidiag", 40, 0, None), ("bidiag", 40, 1, None),
                                                ("z", 40, 1, None), ("z", 10, 1, "1"),
                                                ("bidiag", 5, 0, "1"), ("bidiag", 40, 0, "0")])
def test_approximate_leaves_on_tensor_cores(monkeypatch, name, J, depth, force):
    """Issue-bound approximate plans (many Givens layers) run their approximate leaves as
    densified tcgen05 leaves (the same linear map U_hat_l, multiplied out); GFT_APPROX_TC=1/0
    forces the choice.  Either way the result is the approximate oracle's U_hat^T x."""
    s, d, w = workloads.bidiag_grid() if name == "bidiag" else workloads.z_grid()
    L = oracle.laplacian(64, s, d, w)
    phi = PHI[name] if depth else None
    if force is not None:
        monkeypatch.setenv("GFT_APPROX_TC", force)
    plan = G.Plan(64, s, d, w, None, phi, dtypes=("f32",), max_depth=depth, approx_layers=J,
                  no_cubin_cache=force is not None)
    monkeypatch.delenv("GFT_APPROX_TC", raising=False)
    on_tc = "tc" in plan.kernel_name(G.K_FAST_FWD, "f32").split("_")[1]
    assert on_tc == (force != "0"), plan.kernel_name(G.K_FAST_FWD, "f32")
    if depth == 0:
        _, _, U_o, lam_o = oracle.truncated_jacobi(L, J)
    else:
        lam_o, U_o = oracle.haar_approx_basis(L, phi, J)
    X = torch.randn(4099, 64, generator=torch.Generator().manual_seed(J + depth))
    Y = plan.forward(X.cuda())
    Xr = plan.inverse(Y)
    torch.cuda.synchronize()
    R = oracle.cluster_rotation(U_o, plan.basis(), lam_o)
    e = oracle.aligned_error(Y.cpu().numpy(), oracle.forward(X.numpy(), U_o), R)
    assert e.max() <= 1e-5, e.max()
    assert oracle.relative_error(Xr.cpu().numpy(), X.numpy()).max() <= 2e-5
