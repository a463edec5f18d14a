"""Plain, slow, obviously-correct CPU oracle for the graph Fourier transform.

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this module.  It shares no code with
the library (paper_1907_07875_b200/, include/) and imports nothing from it.

What it computes (Lu & Ortega, arXiv 1907.07875).  The fast GFT is exact
(PAPER.md:79, 81), so the oracle is the plain definition:
  * Laplacian L = D - W + S with l_ii = s_i + sum_{j!=i} w_ij, l_ij = -w_ij
    (eq:def_laplacian / eq:l_from_sw);
  * GFT basis U = eigenvectors of L, ordered by ascending eigenvalue ("graph
    frequencies"), computed with cyclic-by-row Jacobi in fp64;
  * column signs canonicalised: first entry with |u_i| > 1e-8 made positive
    (reading A-3; the paper leaves the sign free);
  * forward Y = X U (row b: y_b = U^T x_b, "projection of x onto u_i")
    and inverse X = Y U^T, in fp64.
Because any orthonormal basis of a repeated eigenspace is a valid GFT,
comparisons are made per eigenvalue cluster (reading A-4/A-5).

Also here, for pinning the library's decomposition (Theorem 3/4): the permuted
butterfly matrix B_phi (eq:B_phi) and the conjugation
B_phi^T L B_phi (eq:BLB), both as plain matrix products.

Pins (tests/test_oracle.py): DCT-II closed form for the uniform line,
the printed C4 GFT matrix (tests/golden/c4_gft.txt), DFT bin
energies for the cycle, 2D-DCT eigenvalues for the uniform grid
(PAPER.md:639), LAPACK eigh cross-check, quadratic form eq:lqf, Parseval,
orthonormality, residual, B_{n,p} structure (eq:Bnp).
"""
from __future__ import annotations

import math

import numpy as np

SIGN_TOL = 1e-8          # reading A-3
CLUSTER_RTOL = 1e-9      # reading A-5


# ---------------------------------------------------------------------------
# Graph -> Laplacian  (eq:def_laplacian, eq:l_from_sw)
# ---------------------------------------------------------------------------
def laplacian(n, src, dst, w, self_loops=None):
    """Dense L: l_ij = -w_ij (i != j), l_ii = s_i + sum_{j != i} w_ij.
    Each self-loop is counted once (reading A-1)."""
    L = np.zeros((n, n), dtype=np.float64)
    for i, j, wt in zip(src, dst, w):
        i, j, wt = int(i), int(j), float(wt)
        if i == j:
            raise ValueError("self-edge in edge list; self-loops go in self_loops")
        L[i, j] -= wt
        L[j, i] -= wt
        L[i, i] += wt
        L[j, j] += wt
    if self_loops is not None:
        for i in range(n):
            L[i, i] += float(self_loops[i])
    return L


def normalized_laplacian(L):
    """Symmetric normalised Laplacian D^{-1/2} L D^{-1/2} with
    d_i = sum_j w_ij, w_ii = s_i, which equals the diagonal l_ii."""
    d = np.diag(L).astype(np.float64)
    if np.any(d <= 0):
        raise ValueError("normalized Laplacian needs positive degrees")
    r = 1.0 / np.sqrt(d)
    return L * r[:, None] * r[None, :]


def quadratic_form_edges(n, src, dst, w, self_loops, f):
    """f^T L f evaluated edge by edge: sum_e w (f_i - f_j)^2 + sum_k s_k f_k^2 (eq:lqf)."""
    tot = 0.0
    for i, j, wt in zip(src, dst, w):
        tot += float(wt) * (f[int(i)] - f[int(j)]) ** 2
    if self_loops is not None:
        tot += float(np.sum(np.asarray(self_loops) * np.asarray(f) ** 2))
    return tot


# ---------------------------------------------------------------------------
# Cyclic-by-row Jacobi eigensolver (fp64).  Not in the paper (SPEC.md:285 calls it
# plumbing); it is the classical Givens-rotation diagonalisation, cf. eq:givens
# applied until convergence.
# ---------------------------------------------------------------------------
def jacobi_eigh(A, tol=1e-15, max_sweeps=100):
    A = np.array(A, dtype=np.float64, copy=True)
    n = A.shape[0]
    if not np.allclose(A, A.T, rtol=0, atol=1e-12 * max(1.0, np.abs(A).max(initial=0.0))):
        raise ValueError("matrix not symmetric")
    V = np.eye(n)
    fro = np.linalg.norm(A)
    for _ in range(max_sweeps):
        off = math.sqrt(float(np.sum((A - np.diag(np.diag(A))) ** 2)))
        if off <= tol * fro or off == 0.0:
            break
        rotated = False
        for p in range(n - 1):
            for q in range(p + 1, n):
                apq = A[p, q]
                if apq == 0.0:
                    continue
                if abs(apq) <= 1e-300:
                    continue
                tau = (A[q, q] - A[p, p]) / (2.0 * apq)
                if abs(tau) > 1e150:          # tau^2 would overflow: t -> 1/(2 tau)
                    t = 1.0 / (2.0 * tau)
                else:
                    t = (1.0 if tau >= 0 else -1.0) / (abs(tau) + math.sqrt(1.0 + tau * tau))
                c = 1.0 / math.sqrt(1.0 + t * t)
                s = t * c
                # A <- J^T A J with J = [[c, s], [-s, c]] in the (p, q) plane
                cp, cq = A[:, p].copy(), A[:, q].copy()
                A[:, p] = c * cp - s * cq
                A[:, q] = s * cp + c * cq
                rp, rq = A[p, :].copy(), A[q, :].copy()
                A[p, :] = c * rp - s * rq
                A[q, :] = s * rp + c * rq
                A[p, q] = A[q, p] = 0.0
                vp, vq = V[:, p].copy(), V[:, q].copy()
                V[:, p] = c * vp - s * vq
                V[:, q] = s * vp + c * vq
                rotated = True
        if not rotated:
            break
    else:
        raise RuntimeError("Jacobi did not converge")
    return np.diag(A).copy(), V


def canonicalize_signs(U, tol=SIGN_TOL):
    """First entry with |u_i| > tol made positive, column by column (reading A-3)."""
    U = U.copy()
    for k in range(U.shape[1]):
        col = U[:, k]
        idx = np.flatnonzero(np.abs(col) > tol)
        if idx.size and col[idx[0]] < 0:
            U[:, k] = -col
    return U


def gft_basis(L):
    """(lambda ascending, canonical U) of the Laplacian L."""
    lam, V = jacobi_eigh(L)
    order = np.argsort(lam, kind="stable")
    lam = lam[order]
    U = canonicalize_signs(V[:, order])
    return lam, U


def gft_basis_of_graph(n, src, dst, w, self_loops=None):
    return gft_basis(laplacian(n, src, dst, w, self_loops))


# ---------------------------------------------------------------------------
# Dense transforms (the "matrix GFT") in fp64
# ---------------------------------------------------------------------------
def forward(X, U):
    """Y = X U: row b holds U^T x_b, coefficients in ascending-eigenvalue order."""
    return np.asarray(X, dtype=np.float64) @ U


def inverse(Y, U):
    """X = Y U^T: row b holds U y_b."""
    return np.asarray(Y, dtype=np.float64) @ U.T


def graph_filter(X, U, h):
    """Graph spectral filtering: row b -> U diag(h) U^T x_b, i.e. X U diag(h) U^T."""
    return ((np.asarray(X, dtype=np.float64) @ U) * np.asarray(h, dtype=np.float64)) @ U.T


def forward_rows_loop(X, U):
    """Same as forward() but a plain per-row loop (used to time a bounded sample the
    way the paper's C 'matrix GFT' runs: one n x n matrix-vector product per signal)."""
    X = np.asarray(X, dtype=np.float64)
    out = np.empty_like(X)
    Ut = U.T.copy()
    for b in range(X.shape[0]):
        out[b] = Ut @ X[b]
    return out


# ---------------------------------------------------------------------------
# Eigen-clusters and per-cluster comparison (readings A-4, A-5, A-17)
# ---------------------------------------------------------------------------
def clusters(lam, rtol=CLUSTER_RTOL):
    lam = np.asarray(lam)
    tol = rtol * max(1.0, float(np.max(np.abs(lam))) if lam.size else 1.0)
    out, start = [], 0
    for k in range(1, len(lam) + 1):
        if k == len(lam) or lam[k] - lam[k - 1] > tol:
            out.append(list(range(start, k)))
            start = k
    return out


def cluster_rotation(U_o, U_f, lam):
    """R = blockdiag_C U_o[:,C]^T U_f[:,C]; orthogonal iff U_f spans the same eigenspaces."""
    n = U_o.shape[0]
    R = np.zeros((n, n))
    for C in clusters(lam):
        R[np.ix_(C, C)] = U_o[:, C].T @ U_f[:, C]
    return R


def aligned_error(Y_hat, Y_ref, R):
    """e_b = ||Y_hat_b R^T - Y_b|| / ||Y_b|| per signal (fp64)."""
    Y_hat = np.asarray(Y_hat, dtype=np.float64)
    Y_ref = np.asarray(Y_ref, dtype=np.float64)
    d = Y_hat @ R.T - Y_ref
    return np.linalg.norm(d, axis=1) / np.maximum(np.linalg.norm(Y_ref, axis=1), 1e-300)


def energy_error(Y_hat, Y_ref, lam):
    """e'_b = sqrt(sum_C (||Y_hat_{b,C}|| - ||Y_{b,C}||)^2) / ||Y_b||  (basis-free)."""
    Y_hat = np.asarray(Y_hat, dtype=np.float64)
    Y_ref = np.asarray(Y_ref, dtype=np.float64)
    acc = np.zeros(Y_ref.shape[0])
    for C in clusters(lam):
        acc += (np.linalg.norm(Y_hat[:, C], axis=1) - np.linalg.norm(Y_ref[:, C], axis=1)) ** 2
    return np.sqrt(acc) / np.maximum(np.linalg.norm(Y_ref, axis=1), 1e-300)


def relative_error(A, B):
    """Per-row relative L2 error ||A_b - B_b|| / ||B_b||."""
    A = np.asarray(A, dtype=np.float64)
    B = np.asarray(B, dtype=np.float64)
    return np.linalg.norm(A - B, axis=1) / np.maximum(np.linalg.norm(B, axis=1), 1e-300)


# ---------------------------------------------------------------------------
# Butterfly matrices, for pinning the library's decomposition
# ---------------------------------------------------------------------------
def butterfly_Bnp(n, p):
    """B_{n,p} of eq:Bnp, 0-based: pairs i <-> n-1-i for i < p."""
    B = np.zeros((n, n))
    r = 1.0 / math.sqrt(2.0)
    for i in range(n):
        if i < p:
            B[i, i] = r
            B[i, n - 1 - i] = r
        elif i >= n - p:
            B[i, i] = -r
            B[i, n - 1 - i] = r
        else:
            B[i, i] = 1.0
    return B


def butterfly_Bphi(phi):
    """B_phi of eq:B_phi; V_X = smaller index of each pair (A-6)."""
    phi = np.asarray(phi)
    n = len(phi)
    B = np.zeros((n, n))
    r = 1.0 / math.sqrt(2.0)
    for i in range(n):
        j = int(phi[i])
        if j == i:
            B[i, i] = 1.0                      # V_Z
        elif i < j:                            # i in V_X
            B[i, i] = r
            B[i, j] = r
        else:                                  # i in V_Y
            B[i, i] = -r
            B[i, j] = r
    return B


def partition(phi):
    """(V_X, V_Y, V_Z) with V_X the smaller index of each pair (A-6)."""
    phi = np.asarray(phi)
    vx = [i for i in range(len(phi)) if phi[i] > i]
    vy = [int(phi[i]) for i in vx]
    vz = [i for i in range(len(phi)) if phi[i] == i]
    return vx, vy, vz


def conjugated_laplacian(L, phi):
    """L_phi = B_phi^T L B_phi by plain matrix products."""
    B = butterfly_Bphi(phi)
    return B.T @ L @ B


def decompose_blocks(L, phi):
    """(L+, L-) read off B_phi^T L B_phi: L+ on V_X then V_Z (in that order), L- on V_Y
    ordered as phi(V_X) (Theorem 3 / eq:blkdiag_G)."""
    G = conjugated_laplacian(L, phi)
    vx, vy, vz = partition(phi)
    plus = vx + vz
    return G[np.ix_(plus, plus)], G[np.ix_(vy, vy)], G, (vx, vy, vz)
