"""Pins of the approximate-GFT oracle (NEXT-4) -- -m "not gpu".

Each pin is fixed by mathematics, not by the oracle's own code: Jacobi's invariant
off(G^T A G)^2 = off(A)^2 - 2 a_pq^2, exact diagonalisation of a 2x2 by one rotation, the
J = 0 permutation, convergence of many layers to the exact GFT (distinct eigenvalues, as the
paper states for both test graphs), and closed forms of delta / epsilon."""
import math

import numpy as np
import pytest

import oracle
import workloads


def test_two_by_two_one_rotation_is_exact():
    rng = np.random.default_rng(0)
    for _ in range(20):
        a, b, c = rng.uniform(-2, 2, 3)
        L = np.array([[a, b], [b, c]])
        layers, perm, Uh, lam = oracle.truncated_jacobi(L, 1)
        assert len(layers) == 1 and len(layers[0]) == 1
        ref = np.linalg.eigvalsh(L)                      # library routine, independent
        assert np.abs(lam - ref).max() < 1e-14 * max(1, abs(L).max())
        assert np.abs(Uh.T @ L @ Uh - np.diag(lam)).max() < 1e-14 * max(1, abs(L).max())


def test_zero_layers_is_the_sorting_permutation():
    s, d, w = workloads.bidiag_grid()
    L = oracle.laplacian(64, s, d, w)
    layers, perm, Uh, lam = oracle.truncated_jacobi(L, 0)
    assert layers == []
    assert np.array_equal(Uh, np.eye(64)[:, perm])
    assert np.array_equal(lam, np.sort(np.diag(L), kind="stable"))


def test_layers_are_disjoint_and_jacobi_invariant_holds():
    s, d, w = workloads.z_grid()
    L = oracle.laplacian(64, s, d, w)
    trace = []
    layers, perm, Uh, lam = oracle.truncated_jacobi(L, 12, trace=trace)
    assert len(layers) == 12
    A = L.copy()
    k = 0
    for layer in layers:
        idx = [i for p, q, _, _ in layer for i in (p, q)]
        assert len(idx) == len(set(idx))                 # disjoint pairs in a layer
        G = oracle.givens_matrix(64, layer)
        assert np.abs(G.T @ G - np.eye(64)).max() < 1e-14
        before = oracle.off2(A)
        drop = sum(2 * tr[1] ** 2 for tr in trace[k:k + len(layer)])
        k += len(layer)
        A = G.T @ A @ G
        # rotations in a layer touch disjoint rows/cols: the layer removes 2 sum a_pq^2
        assert abs(before - drop - oracle.off2(A)) < 1e-11 * before
    # U_hat realises the accumulated rotations, columns sorted by the final diagonal
    assert np.abs(Uh.T @ L @ Uh - (A[np.ix_(perm, perm)])).max() < 1e-11
    assert np.abs(Uh.T @ Uh - np.eye(64)).max() < 1e-13
    assert np.all(np.diff(lam) >= 0)


@pytest.mark.parametrize("graph", ["bidiag", "z"])
def test_many_layers_converge_to_the_exact_gft(graph):
    s, d, w = workloads.bidiag_grid() if graph == "bidiag" else workloads.z_grid()
    L = oracle.laplacian(64, s, d, w)
    lam_o, U_o = oracle.gft_basis(L)
    layers, perm, Uh, lam = oracle.truncated_jacobi(L, 400)
    assert np.abs(lam - lam_o).max() < 1e-10
    assert oracle.delta_error(Uh, U_o) < 1e-7
    # the trend of Fig. 10: delta drops as layers are added
    deltas = [oracle.delta_error(oracle.truncated_jacobi(L, J)[2], U_o) for J in (0, 10, 20, 40, 80)]
    assert all(b < a for a, b in zip(deltas, deltas[1:])), deltas


def test_delta_and_epsilon_closed_forms():
    rng = np.random.default_rng(4)
    n = 9
    U, _ = np.linalg.qr(rng.normal(size=(n, n)))
    X = rng.normal(size=(50, n))
    assert oracle.delta_error(U, U) < 1e-14
    assert oracle.delta_error(-U, U) < 1e-14                  # "avoid this sign ambiguity"
    assert oracle.epsilon_error(-U, U, X) < 1e-24
    P = U.copy()
    P[:, [2, 5]] = P[:, [5, 2]]
    # |P^T U| - I has four unit entries: ||.||_F = 2
    assert abs(oracle.delta_error(P, U) - 2 / math.sqrt(n)) < 1e-13
    # epsilon of the swap: per signal (|y2|-|y5|)^2 twice
    Y = X @ U
    ref = float(np.mean(2 * (np.abs(Y[:, 2]) - np.abs(Y[:, 5])) ** 2))
    assert abs(oracle.epsilon_error(P, U, X) - ref) < 1e-12


def test_haar_approx_basis_limits():
    """J large -> the exact GFT; any J -> orthogonal and the B_phi structure kept."""
    s, d, w = workloads.bidiag_grid()
    L = oracle.laplacian(64, s, d, w)
    phi = np.array([8 * (i % 8) + i // 8 for i in range(64)])     # transpose (main diagonal)
    assert np.abs(L - L[np.ix_(phi, phi)]).max() == 0
    lam_o, U_o = oracle.gft_basis(L)
    lam, Uh = oracle.haar_approx_basis(L, phi, 300)
    assert np.abs(lam - lam_o).max() < 1e-10
    assert oracle.delta_error(Uh, U_o) < 1e-7
    for J in (0, 5, 20):
        lam, Uh = oracle.haar_approx_basis(L, phi, J)
        assert np.abs(Uh.T @ Uh - np.eye(64)).max() < 1e-13
        # every column is even or odd under phi (a Haar-stage output)
        Jphi = np.eye(64)[phi]
        par = np.einsum("ik,ik->k", Uh, Jphi @ Uh)
        assert np.all(np.abs(np.abs(par) - 1) < 1e-12)
    # Haar + approximate converges faster than approximate alone
    # (delta is dominated by mis-ordered columns for J <~ 10 on both, so compare J >= 20)
    for J in (20, 30, 40, 60):
        d_h = oracle.delta_error(oracle.haar_approx_basis(L, phi, J)[1], U_o)
        d_a = oracle.delta_error(oracle.truncated_jacobi(L, J)[2], U_o)
        assert d_h < d_a, (J, d_h, d_a)
