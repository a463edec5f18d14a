"""Pins for the CPU oracle (-m "not gpu").  Each test checks the oracle against something
the paper or mathematics fixes independently of the oracle's own code path."""
import math

import numpy as np
import pytest

import oracle
import workloads
from conftest import read_golden


def _proj(U, cols):
    Q = U[:, cols]
    return Q @ Q.T


# --- Laplacian (eq:l_from_sw PAPER.md:122-123; eq:lqf PAPER.md:130-133) -------------
def test_laplacian_small_examples():
    # P2, w=1 -> [[1,-1],[-1,1]]  (by hand from eq:l_from_sw)
    L = oracle.laplacian(2, [0], [1], [1.0])
    assert np.array_equal(L, [[1, -1], [-1, 1]])
    # edge 1 with self-loops 2,2 -> [[3,-1],[-1,3]]  (each loop counted once, A-1)
    L = oracle.laplacian(2, [0], [1], [1.0], [2.0, 2.0])
    assert np.array_equal(L, [[3, -1], [-1, 3]])
    # row sums equal self-loops (eq:sw_from_l)
    rng = np.random.default_rng(0)
    s, d, w, loops, _ = workloads.random_symmetric_graph(rng, 9)
    L = oracle.laplacian(9, s, d, w, loops)
    assert np.allclose(L.sum(axis=1), loops, atol=1e-13)


def test_quadratic_form_matches_edge_sum():
    rng = np.random.default_rng(1)
    for n in (2, 5, 13):
        s, d, w, loops, _ = workloads.random_symmetric_graph(rng, n, negative=True)
        L = oracle.laplacian(n, s, d, w, loops)
        for _ in range(5):
            f = rng.standard_normal(n)
            q1 = f @ L @ f
            q2 = oracle.quadratic_form_edges(n, s, d, w, loops, f)
            assert abs(q1 - q2) <= 1e-12 * max(1.0, abs(q2))
    # P2 f=(1,-1) -> 4 ; C4 f=(1,0,-1,0) -> 4
    assert oracle.quadratic_form_edges(2, [0], [1], [1.0], None, [1.0, -1.0]) == 4.0
    s, d, w = workloads.cycle_graph(4)
    assert oracle.quadratic_form_edges(4, s, d, w, None, [1.0, 0, -1.0, 0]) == 4.0


# --- Jacobi vs LAPACK (library routine) ------------------------------------------------
@pytest.mark.parametrize("n", [1, 2, 3, 7, 16, 40])
def test_jacobi_matches_lapack(n):
    rng = np.random.default_rng(n)
    A = rng.standard_normal((n, n)); A = A + A.T
    lam, V = oracle.jacobi_eigh(A)
    ref = np.linalg.eigh(A)[0]
    assert np.allclose(np.sort(lam), ref, atol=1e-12 * max(1, np.abs(ref).max()))
    assert np.abs(V.T @ V - np.eye(n)).max() < 1e-13
    assert np.abs(A @ V - V * lam).max() < 1e-11


def test_jacobi_degenerate_matrix():
    # A = Q diag(1,1,1,3,3,5) Q^T: eigenspaces must match LAPACK's projectors
    rng = np.random.default_rng(7)
    Q, _ = np.linalg.qr(rng.standard_normal((6, 6)))
    A = Q @ np.diag([1, 1, 1, 3, 3, 5.0]) @ Q.T
    lam, U = oracle.gft_basis(A)
    assert np.allclose(lam, [1, 1, 1, 3, 3, 5], atol=1e-12)
    for C in ([0, 1, 2], [3, 4], [5]):
        assert np.abs(_proj(U, C) - _proj(Q, C)).max() < 1e-12


def test_jacobi_rejects_asymmetric():
    with pytest.raises(ValueError):
        oracle.jacobi_eigh(np.array([[1.0, 2.0], [0.0, 1.0]]))


# --- Closed forms ----------------------------------------------------------------------
@pytest.mark.parametrize("n", [4, 8, 16])
def test_uniform_line_is_dct2(n):
    """Uniform line graph GFT = DCT-II: u_k(i) = c_k cos(pi k (i+1/2)/n),
    lambda_k = 2 - 2 cos(pi k / n).  All eigenvalues simple; DCT signs are canonical."""
    s, d, w = workloads.path_graph(n)
    lam, U = oracle.gft_basis_of_graph(n, s, d, w)
    k = np.arange(n)
    assert np.abs(lam - (2 - 2 * np.cos(np.pi * k / n))).max() < 1e-13
    i = np.arange(n)[:, None]
    C = np.cos(np.pi * k[None, :] * (i + 0.5) / n) * np.where(k == 0, math.sqrt(1 / n), math.sqrt(2 / n))
    assert np.abs(U - C).max() < 1e-12


def test_c4_printed_matrix():
    """U_{C4} printed at PAPER.md:186-194 with eigenvalues (0,2,2,4)."""
    scale, M, lam_g = read_golden("c4_gft.txt")
    Ug = float(scale[0][0]) * np.array(M, dtype=float)
    lam_g = np.array(lam_g[0], dtype=float)
    s, d, w = workloads.cycle_graph(4)
    lam, U = oracle.gft_basis_of_graph(4, s, d, w)
    assert np.abs(lam - lam_g).max() < 1e-14
    # simple eigenvalues: coefficient-wise, signed (the printed columns are canonical)
    assert np.abs(U[:, 0] - Ug[:, 0]).max() < 1e-14
    assert np.abs(U[:, 3] - Ug[:, 3]).max() < 1e-14
    # repeated eigenvalue 2: same eigenspace
    assert np.abs(_proj(U, [1, 2]) - _proj(Ug, [1, 2])).max() < 1e-14
    # and the printed matrix really diagonalises L (pins the golden fixture itself)
    L = oracle.laplacian(4, s, d, w)
    assert np.abs(L @ Ug - Ug * lam_g).max() < 1e-14


@pytest.mark.parametrize("n", [12, 64, 80])
def test_cycle_cluster_energy_is_dft(n):
    """The DFT is a GFT of the cycle: per-cluster energy of U^T x equals
    (|X_k|^2 + |X_{n-k}|^2)/n from an FFT; lambda_k = 2 - 2 cos(2 pi k / n)."""
    s, d, w = workloads.cycle_graph(n)
    lam, U = oracle.gft_basis_of_graph(n, s, d, w)
    ref = np.sort(2 - 2 * np.cos(2 * np.pi * np.arange(n) / n))
    assert np.abs(lam - ref).max() < 1e-12
    rng = np.random.default_rng(n)
    x = rng.standard_normal((5, n))
    y = oracle.forward(x, U)
    F = np.fft.fft(x, axis=1)
    for C in oracle.clusters(lam):
        lam_c = lam[C[0]]
        bins = [k for k in range(n) if abs(2 - 2 * math.cos(2 * math.pi * k / n) - lam_c) < 1e-9]
        assert len(bins) == len(C)
        e_dft = np.sum(np.abs(F[:, bins]) ** 2, axis=1) / n
        e_gft = np.sum(y[:, C] ** 2, axis=1)
        assert np.abs(e_dft - e_gft).max() < 1e-11 * max(1, e_dft.max())


def test_cycle_lemma1_pairing():
    """Lemma 1: the cycle C64 is 2-regular bipartite, so eigenvalues
    pair as lambda <-> 4 - lambda and (u1; -u2) is an eigenvector (parts = even/odd nodes)."""
    n = 64
    s, d, w = workloads.cycle_graph(n)
    L = oracle.laplacian(n, s, d, w)
    lam, U = oracle.gft_basis(L)
    assert np.abs(np.sort(4 - lam) - lam).max() < 1e-12
    sign = np.where(np.arange(n) % 2 == 0, 1.0, -1.0)
    for k in range(n):
        u2 = U[:, k] * sign
        assert np.abs(L @ u2 - (4 - lam[k]) * u2).max() < 1e-11


def test_grid_is_2d_dct():
    """Uniform 4-connected grid GFT = 2D DCT: lambda = mu_a + mu_b and each
    eigenspace is spanned by the separable DCT-II products with that eigenvalue."""
    R = 8
    s, d, w = workloads.grid_graph(R, R)
    lam, U = oracle.gft_basis_of_graph(R * R, s, d, w)
    k = np.arange(R)
    mu = 2 - 2 * np.cos(np.pi * k / R)
    i = np.arange(R)[:, None]
    D = np.cos(np.pi * k[None, :] * (i + 0.5) / R) * np.where(k == 0, math.sqrt(1 / R), math.sqrt(2 / R))
    lam2 = (mu[:, None] + mu[None, :]).ravel()          # index a*R + b
    basis2 = np.einsum("ra,cb->rcab", D, D).reshape(R * R, R * R)   # node r*R+c, freq a*R+b
    assert np.abs(np.sort(lam2) - lam).max() < 1e-12
    for C in oracle.clusters(lam):
        cols = [f for f in range(R * R) if abs(lam2[f] - lam[C[0]]) < 1e-9]
        assert len(cols) == len(C)
        assert np.abs(_proj(U, C) - _proj(basis2, cols)).max() < 1e-11


# --- Invariants on the BASELINE configs -----------------------------------------------
@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg2b", "cfg3", "cfg4", "cfg5a", "cfg5b"])
def test_config_basis_invariants(name):
    cfg = workloads.config(name)
    L = oracle.laplacian(cfg.n, *cfg.edges, cfg.self_loops)
    lam, U = oracle.gft_basis(L)
    assert np.abs(L @ U - U * lam).max() < 1e-10            # north-star residual bound
    assert np.abs(U.T @ U - np.eye(cfg.n)).max() < 1e-12
    assert np.all(np.diff(lam) >= -1e-12)
    ref, V_ref = np.linalg.eigh(L)
    assert np.abs(lam - ref).max() < 1e-11 * max(1, ref.max())
    # eigenspaces vs LAPACK (a routine independent of the oracle's Jacobi), per cluster
    for C in oracle.clusters(lam):
        assert np.abs(_proj(U, C) - _proj(V_ref, C)).max() < 1e-10
    # Theorem 3: spec(L) = spec(L+) u spec(L-) for the config's involution, by LAPACK
    if cfg.phi is not None:
        Lp, Lm, _, _ = oracle.decompose_blocks(L, cfg.phi)
        spec = np.sort(np.concatenate([np.linalg.eigvalsh(Lp), np.linalg.eigvalsh(Lm)]))
        assert np.abs(spec - ref).max() < 1e-11 * max(1, ref.max())
    # Parseval ||U^T x|| = ||x||
    x = workloads.signals(cfg, batch=64, dtype="f64").numpy()
    y = oracle.forward(x, U)
    assert np.abs(np.linalg.norm(y, axis=1) / np.linalg.norm(x, axis=1) - 1).max() < 1e-13
    assert np.abs(oracle.inverse(y, U) - x).max() < 1e-12 * np.abs(x).max()
    # loop form of the dense transform agrees with the matmul form
    assert np.abs(oracle.forward_rows_loop(x[:8], U) - y[:8]).max() < 1e-12


# --- Butterfly matrices (eq:Bnp, eq:B_phi, Theorem 3) ----------------------------------
def test_bnp_structure():
    for n, p in ((4, 2), (8, 3), (7, 3), (5, 0)):
        B = oracle.butterfly_Bnp(n, p)
        assert np.allclose(B, B.T) and np.allclose(B @ B.T, np.eye(n), atol=1e-15)
        x = np.arange(1.0, n + 1)
        y = B @ x
        r = 1 / math.sqrt(2)
        for i in range(n):      # PAPER.md:209-212 (1-based there)
            if i < p:
                assert abs(y[i] - r * (x[i] + x[n - 1 - i])) < 1e-14
            elif i >= n - p:
                assert abs(y[i] - r * (-x[i] + x[n - 1 - i])) < 1e-14
            else:
                assert y[i] == x[i]
        # reversal phi restricted to first p pairs gives the same matrix
        phi = np.arange(n)
        for i in range(p):
            phi[i], phi[n - 1 - i] = n - 1 - i, i
        assert np.allclose(oracle.butterfly_Bphi(phi), B)


def test_c4_decomposition_example():
    """C4 with phi=(3,2,1,0): G+ = path w=1 (no loops), G- = edge 1 with loops 2,2
    (by hand from Theorem 4)."""
    s, d, w = workloads.cycle_graph(4)
    L = oracle.laplacian(4, s, d, w)
    Lp, Lm, G, _ = oracle.decompose_blocks(L, [3, 2, 1, 0])
    assert np.allclose(Lp, [[1, -1], [-1, 1]], atol=1e-15)
    assert np.allclose(Lm, [[3, -1], [-1, 3]], atol=1e-15)


def test_theorem3_offblocks_random():
    rng = np.random.default_rng(3)
    for trial in range(50):
        n = int(rng.integers(2, 14))
        s, d, w, loops, phi = workloads.random_symmetric_graph(rng, n, negative=bool(trial % 2))
        L = oracle.laplacian(n, s, d, w, loops)
        G = oracle.conjugated_laplacian(L, phi)
        vx, vy, vz = oracle.partition(phi)
        assert np.abs(G[np.ix_(vx + vz, vy)]).max(initial=0) < 1e-13 * max(1, np.abs(L).max())
        # spectrum preserved (orthogonal similarity)
        Lp, Lm, _, _ = oracle.decompose_blocks(L, phi)
        spec = np.sort(np.concatenate([np.linalg.eigvalsh(Lp) if Lp.size else [],
                                       np.linalg.eigvalsh(Lm) if Lm.size else []]))
        assert np.abs(spec - np.linalg.eigvalsh(L)).max() < 1e-11
    # converse: breaking symmetry breaks the off-block (Lemma 3 'only if')
    s, d, w = workloads.path_graph(6)
    w = w.copy(); w[0] *= 1.01
    L = oracle.laplacian(6, s, d, w)
    G = oracle.conjugated_laplacian(L, [5, 4, 3, 2, 1, 0])
    assert np.abs(G[np.ix_([0, 1, 2], [3, 4, 5])]).max() > 1e-4


def test_normalized_laplacian_pins():
    """D^{-1/2} L D^{-1/2}: for a k-regular loop-free graph it is L/k (the
    cycle C12 is 2-regular); for a bipartite graph its spectrum is symmetric about 1
    (lambda <-> 2 - lambda, the normalised counterpart of Lemma 1 / Theorem 2)."""
    s, d, w = workloads.cycle_graph(12)
    L = oracle.laplacian(12, s, d, w)
    N = oracle.normalized_laplacian(L)
    assert np.abs(N - L / 2).max() < 1e-15
    rng = np.random.default_rng(4)
    pairs = [(a, 6 + b) for a in range(6) for b in range(7) if rng.random() < 0.6]
    pairs += [(a, 6 + a) for a in range(6)]                     # keep it connected-ish
    pairs = sorted(set(pairs))
    s = np.array([p[0] for p in pairs]); d = np.array([p[1] for p in pairs])
    w = rng.uniform(0.5, 2.0, len(pairs))
    L = oracle.laplacian(13, s, d, w)
    lam, U = oracle.gft_basis(oracle.normalized_laplacian(L))
    assert np.abs(np.sort(2 - lam) - lam).max() < 1e-12
    assert np.abs(lam).min() < 1e-12                              # D^{1/2} 1 is in the kernel
    with pytest.raises(ValueError):
        oracle.normalized_laplacian(np.zeros((2, 2)))


@pytest.mark.parametrize("name", ["cfg3", "cfg4"])
def test_graph_filter_closed_forms(name):
    """U diag(h) U^T: h = 1 -> I, h = lambda -> L, h = lambda^2 -> L^2, h = exp(-t lambda) ->
    expm(-t L) (SciPy's Pade expm, a library routine)."""
    import scipy.linalg
    cfg = workloads.config(name)
    L = oracle.laplacian(cfg.n, *cfg.edges, cfg.self_loops)
    lam, U = oracle.gft_basis(L)
    X = workloads.signals(cfg, batch=32, dtype="f64").numpy()
    assert np.abs(oracle.graph_filter(X, U, np.ones(cfg.n)) - X).max() < 1e-12
    assert np.abs(oracle.graph_filter(X, U, lam) - X @ L).max() < 1e-11
    assert np.abs(oracle.graph_filter(X, U, lam ** 2) - X @ L @ L).max() < 1e-10
    t = 0.3
    assert np.abs(oracle.graph_filter(X, U, np.exp(-t * lam)) - X @ scipy.linalg.expm(-t * L)).max() < 1e-12


def test_cluster_metrics_are_sign_and_rotation_invariant():
    s, d, w = workloads.cycle_graph(8)
    lam, U = oracle.gft_basis_of_graph(8, s, d, w)
    rng = np.random.default_rng(5)
    # rotate inside every 2-fold cluster and flip signs
    Uf = U.copy()
    for C in oracle.clusters(lam):
        if len(C) == 2:
            th = rng.uniform(0, 2 * np.pi)
            R2 = np.array([[np.cos(th), -np.sin(th)], [np.sin(th), np.cos(th)]])
            Uf[:, C] = U[:, C] @ R2
    Uf[:, 0] *= -1
    x = rng.standard_normal((10, 8))
    Yo, Yf = oracle.forward(x, U), oracle.forward(x, Uf)
    R = oracle.cluster_rotation(U, Uf, lam)
    assert oracle.aligned_error(Yf, Yo, R).max() < 1e-14
    assert oracle.energy_error(Yf, Yo, lam).max() < 1e-14
    # a wrong basis (swap columns across clusters) is caught by the energy metric
    Ubad = U.copy(); Ubad[:, [0, 7]] = Ubad[:, [7, 0]]
    assert oracle.energy_error(oracle.forward(x, Ubad), Yo, lam).max() > 1e-2
