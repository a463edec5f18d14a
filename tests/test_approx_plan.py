"""Approximate plans (NEXT-4) on the host, against the approximate oracle
(-m "not gpu").

"Approximate GFT" = max_depth 0 + approx_layers J (the whole graph is one truncated-Jacobi
leaf); "Haar + approximate" = Haar stages, then truncated-Jacobi leaves.  The library's
exported U_hat must equal the oracle's construction (same greedy reading R-4): the pure
approximate basis column for column, the one-stage Haar + approximate basis per cluster of
approximate eigenvalues and up to column sign (the V_X orientation of a pair flips the
signs inside a leaf's Laplacian, which flips realised column signs only)."""
import numpy as np
import pytest

import oracle
import workloads
from paper_1907_07875_b200 import gft as G

GRAPHS = {"bidiag": (workloads.bidiag_grid, np.array([8 * (i % 8) + i // 8 for i in range(64)], np.int32)),
          "z": (workloads.z_grid, np.array([63 - i for i in range(64)], np.int32))}


def _graph(name):
    f, phi = GRAPHS[name]
    s, d, w = f()
    return s, d, w, phi, oracle.laplacian(64, s, d, w)


def _cluster_match(lam_o, U_o, U_f, atol):
    worst = 0.0
    for C in oracle.clusters(lam_o):
        worst = max(worst, np.abs(U_f[:, C] @ U_f[:, C].T - U_o[:, C] @ U_o[:, C].T).max())
    assert worst < atol, worst


@pytest.mark.parametrize("name", ["bidiag", "z"])
@pytest.mark.parametrize("J", [0, 1, 5, 20, 40])
def test_pure_approximate_matches_oracle(name, J):
    s, d, w, phi, L = _graph(name)
    plan = G.Plan(64, s, d, w, host_only=True, max_depth=0, approx_layers=J)
    layers, perm, U_o, lam_o = oracle.truncated_jacobi(L, J)
    info = plan.info()
    assert info["n_approx_leaves"] == 1 and info["depth"] == 0
    nrot = sum(len(l) for l in layers)
    assert info["n_givens"] == nrot
    assert info["adds"] == 2 * nrot and info["mults"] == 2 * nrot + 64
    assert info["paper_mults"] == 4 * nrot
    assert np.abs(plan.eigenvalues() - lam_o).max() < 1e-12
    assert np.abs(plan.basis() - U_o).max() < 1e-12          # same signs: no sign rule
    assert info["orth_error"] < 1e-13


@pytest.mark.parametrize("name", ["bidiag", "z"])
@pytest.mark.parametrize("J", [0, 5, 10, 20, 40])
def test_haar_plus_approximate_matches_oracle(name, J):
    s, d, w, phi, L = _graph(name)
    plan = G.Plan(64, s, d, w, None, phi, host_only=True, max_depth=1, approx_layers=J)
    lam_o, U_o = oracle.haar_approx_basis(L, phi, J)
    assert plan.info()["units_per_level"][0] == int(np.sum(phi > np.arange(64)))
    assert np.abs(plan.eigenvalues() - lam_o).max() < 1e-12
    _cluster_match(lam_o, U_o, plan.basis(), 1e-11)


def test_error_metrics_and_convergence():
    """Paper's observations on the library's plans: delta falls with J,
    Haar + approximate converges faster, and enough layers give the exact GFT."""
    s, d, w, phi, L = _graph("bidiag")
    lam_e, U_e = oracle.gft_basis(L)
    d_a, d_h = [], []
    for J in (5, 20, 40, 80):
        a = G.Plan(64, s, d, w, host_only=True, max_depth=0, approx_layers=J)
        h = G.Plan(64, s, d, w, None, phi, host_only=True, approx_layers=J)   # unlimited depth
        d_a.append(oracle.delta_error(a.basis(), U_e))
        d_h.append(oracle.delta_error(h.basis(), U_e))
        assert h.info()["orth_error"] < 1e-13
    assert all(y < x for x, y in zip(d_a, d_a[1:])), d_a
    assert all(h < a for h, a in zip(d_h[1:], d_a[1:])), (d_h, d_a)
    exact = G.Plan(64, s, d, w, None, phi, host_only=True, approx_layers=400)
    assert oracle.delta_error(exact.basis(), U_e) < 1e-7
    assert np.abs(exact.eigenvalues() - lam_e).max() < 1e-10


def test_approx_min_leaf_and_defaults():
    s, d, w, phi, L = _graph("z")
    exact = G.Plan(64, s, d, w, None, phi, host_only=True)
    assert exact.info()["n_approx_leaves"] == 0 and exact.info()["n_givens"] == 0
    big = G.Plan(64, s, d, w, None, phi, host_only=True, approx_layers=10, approx_min_leaf=100)
    assert big.info()["n_approx_leaves"] == 0
    assert np.abs(big.basis() - exact.basis()).max() == 0
    with pytest.raises(G.GFTError):
        G.Plan(64, s, d, w, host_only=True, approx_layers=-2)


def test_two_by_two_leaf_is_exact_with_one_layer():
    """A 2-node graph: one rotation diagonalises it exactly (the approximate plan equals the
    exact GFT up to column signs)."""
    s = np.array([0], np.int32); d = np.array([1], np.int32); w = np.array([0.7])
    loops = np.array([0.3, 1.1])                    # asymmetric: no involution
    plan = G.Plan(2, s, d, w, loops, host_only=True, approx_layers=1)
    assert plan.info()["n_givens"] == 1
    L = oracle.laplacian(2, s, d, w, loops)
    lam, U = oracle.gft_basis(L)
    assert np.abs(plan.eigenvalues() - lam).max() < 1e-14
    assert np.abs(np.abs(plan.basis()) - np.abs(U)).max() < 1e-14
