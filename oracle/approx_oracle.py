"""Plain CPU oracle of the APPROXIMATE GFTs of the paper's second experiment (NEXT-4).

TEST INFRASTRUCTURE ONLY (same rules as gft_oracle.py): only tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / --impl reference legs may import it; it shares no code with
the library.

What it computes (Sec. VI-B):
  * "Approximate GFT": J layers of parallel Givens rotations found by the parallel truncated
    Jacobi algorithm, "a greedy-based algorithm that progressively approximate U^T L U to a
    diagonal matrix", followed by a final permutation Pi_{J+1}.
    The cited algorithm itself is not in PAPER.md; the layer rule follows the reading of
    SURVEY §8(f) NEXT-4 / DESIGN.md reading R-4:
      each layer: repeatedly take the not-yet-used index pair (p, q) with the largest
      |a_pq| (ties within relative TIE_RTOL -> lexicographically smallest (p, q)), rotate
      with the classical Jacobi angle that annihilates a_pq, until no disjoint pair with
      |a_pq| > ZERO_RTOL * max(1, max|L|) remains (a_pp, a_qq equal within TIE_RTOL take
      the 45 degree rotation); an empty layer ends the iteration;
      Pi_{J+1} sorts the final diagonal ascending (stable).
    The approximate basis is U_hat = G_1 G_2 ... G_J Pi, approximate eigenvalues =
    diag(U_hat^T L U_hat).  Column signs are those the rotations produce (no sign rule: the
    paper's metrics take absolute values).
  * "Haar + approximate GFT": one Haar stage B_phi (eq:B_phi) with the
    sub-GFTs of L+ and L- (Theorem 3 blocks of B_phi^T L B_phi) replaced by their truncated
    Jacobi approximations.
  * the two error metrics: delta (sign-normalised relative error) and
    epsilon (empirical average error).

Pins (tests/test_approx_oracle.py): 2x2 exactly diagonalised by one rotation; J = 0 is the
diagonal-sorting permutation; each rotation lowers off(A)^2 by exactly 2 a_pq^2 (Jacobi's
invariant); many layers converge to the exact GFT (delta -> 0); delta/epsilon closed forms
for U, -U and a column transposition.
"""
from __future__ import annotations

import math

import numpy as np

from .gft_oracle import butterfly_Bphi, decompose_blocks

TIE_RTOL = 1e-12     # reading R-4: near-equal |a_pq| are ties
ZERO_RTOL = 1e-14    # reading R-4: entries below this (relative) are not rotated


def _rotation(app, aqq, apq, tie_rtol=TIE_RTOL):
    """(c, s) of the classical Jacobi rotation annihilating a_pq (stable tan formula).
    Diagonal entries equal within tie_rtol count as equal (tau = 0 -> the 45 degree
    rotation, t = 1): the sign of a rounding-level tau would otherwise flip the rotation
    direction (reading R-4)."""
    if abs(aqq - app) <= tie_rtol * max(abs(app), abs(aqq), abs(apq)):
        return 1.0 / math.sqrt(2.0), 1.0 / math.sqrt(2.0)
    tau = (aqq - app) / (2.0 * apq)
    if abs(tau) > 1e150:
        t = 1.0 / (2.0 * tau)
    else:
        t = (1.0 if tau >= 0 else -1.0) / (abs(tau) + math.sqrt(1.0 + tau * tau))
    c = 1.0 / math.sqrt(1.0 + t * t)
    return c, t * c


def off2(A):
    """Sum of squared off-diagonal entries."""
    A = np.asarray(A, dtype=np.float64)
    return float(np.sum(A * A) - np.sum(np.diag(A) ** 2))


def truncated_jacobi(L, J, tie_rtol=TIE_RTOL, zero_rtol=ZERO_RTOL, trace=None):
    """J layers of parallel Givens rotations (greedy, reading R-4).

    Returns (layers, perm, U_hat, lam_hat): layers[j] = list of (p, q, c, s) with
    G = I except G[p,p] = G[q,q] = c, G[p,q] = s, G[q,p] = -s (A <- G^T A G);
    U_hat = G_1 ... G_J[:, perm]; lam_hat ascending.  `trace`, if a list, receives
    (off2 before, a_pq) per rotation."""
    A = np.array(L, dtype=np.float64, copy=True)
    n = A.shape[0]
    zt = zero_rtol * max(1.0, float(np.abs(A).max(initial=0.0)))
    V = np.eye(n)
    layers = []
    iu = np.triu_indices(n, 1)
    for _ in range(J):
        used = np.zeros(n, dtype=bool)
        rots = []
        while True:
            free = ~used[iu[0]] & ~used[iu[1]]
            if not free.any():
                break
            vals = np.abs(A[iu])
            vals = np.where(free, vals, -1.0)
            m = float(vals.max())
            if m <= zt:
                break
            k = int(np.flatnonzero(vals >= m * (1.0 - tie_rtol))[0])   # lexicographic first
            p, q = int(iu[0][k]), int(iu[1][k])
            apq = A[p, q]
            if trace is not None:
                trace.append((off2(A), apq))
            c, s = _rotation(A[p, p], A[q, q], apq)
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
            used[p] = used[q] = True
            rots.append((p, q, c, s))
        if not rots:
            break
        layers.append(rots)
    lam = np.diag(A).copy()
    perm = np.argsort(lam, kind="stable")
    return layers, perm, V[:, perm], lam[perm]


def givens_matrix(n, layer):
    """The orthogonal matrix of one layer (product of its disjoint rotations)."""
    G = np.eye(n)
    for p, q, c, s in layer:
        G[p, p] = c
        G[q, q] = c
        G[p, q] = s
        G[q, p] = -s
    return G


def haar_approx_basis(L, phi, J, min_leaf=2):
    """Haar + approximate GFT: one Haar stage from phi (V_X = smaller index
    of each pair), then the truncated-Jacobi approximation of the sub-GFT of each block
    (L+ on V_X then V_Z, L- on phi(V_X)); blocks smaller than min_leaf use the exact
    eigendecomposition.  Columns ordered by approximate eigenvalue (stable).  Returns
    (lam_hat, U_hat)."""
    from .gft_oracle import jacobi_eigh
    Lp, Lm, _, (vx, vy, vz) = decompose_blocks(L, phi)
    B = butterfly_Bphi(phi)
    n = L.shape[0]
    cols, lams = [], []
    for nodes, Lb in ((vx + vz, Lp), (vy, Lm)):
        k = len(nodes)
        if k == 0:
            continue
        if k >= min_leaf:
            _, _, Ub, lb = truncated_jacobi(Lb, J)
        else:
            lb, Ub = jacobi_eigh(Lb)
        E = np.zeros((n, k))
        E[nodes, :] = Ub
        cols.append(B @ E)
        lams.append(lb)
    U = np.concatenate(cols, axis=1)
    lam = np.concatenate(lams)
    order = np.argsort(lam, kind="stable")
    return lam[order], U[:, order]


def delta_error(U_hat, U):
    """delta = ||  |U_hat^T U| - I ||_F / sqrt(n)."""
    U_hat = np.asarray(U_hat, dtype=np.float64)
    U = np.asarray(U, dtype=np.float64)
    n = U.shape[0]
    return float(np.linalg.norm(np.abs(U_hat.T @ U) - np.eye(n)) / math.sqrt(n))


def epsilon_error(U_hat, U, X):
    """epsilon = (1/M) sum_i sum_j (|u_j^T x_i| - |u_hat_j^T x_i|)^2;
    X holds the M signals as rows."""
    X = np.asarray(X, dtype=np.float64)
    d = np.abs(X @ U) - np.abs(X @ U_hat)
    return float(np.sum(d * d) / X.shape[0])
