"""Right Haar stages (NEXT-2, eq:right_gft / eq:right_pm, Lemma 1,
Theorems 1-2) on the host planner, checked against the oracle (-m "not gpu").

A symmetry-free bipartite (sub)graph whose Laplacian has a constant diagonal c -- a
weighted k-regular bipartite graph (Theorem 1) or the normalised Laplacian of any bipartite
graph (Theorem 2) -- is planned as two dense leaves E (part S1) and F (part S2) followed by
min(|S1|, |S2|) coefficient butterflies.  The realised basis must still be THE GFT of the
graph (oracle eigenbasis, per cluster), and the operation count must drop from
n(n-1) adds / n^2 mults to |S1|(|S1|-1) + |S2|(|S2|-1) + 2p adds / |S1|^2 + |S2|^2 mults."""
import numpy as np
import pytest

import oracle
import workloads
from paper_1907_07875_b200 import gft as G


def _proj(U, cols):
    Q = U[:, cols]
    return Q @ Q.T


def _check_basis(L, plan, atol=1e-10):
    lam_o, U_o = oracle.gft_basis(L)
    lam_f, U_f = plan.eigenvalues(), plan.basis()
    n = L.shape[0]
    scale = max(1.0, np.abs(L).max())
    assert np.abs(lam_f - lam_o).max() < 1e-11 * scale
    assert np.abs(L @ U_f - U_f * lam_f).max() < 1e-11 * scale
    assert np.abs(U_f.T @ U_f - np.eye(n)).max() < 1e-12
    for C in oracle.clusters(lam_o):
        if len(C) == 1:
            assert np.abs(U_f[:, C[0]] - U_o[:, C[0]]).max() < atol
        else:
            assert np.abs(_proj(U_f, C) - _proj(U_o, C)).max() < atol
    return lam_o, U_o, U_f


def test_lemma1_pairing_on_oracle_basis():
    """Lemma 1 pinned on the oracle itself: for a weighted k-RBG, if
    (u1; u2) is an eigenvector with eigenvalue lambda then (u1; -u2) is one with 2k - lambda.
    Theorem 2's analogue holds for the normalised Laplacian of any bipartite graph (c = 1)."""
    rng = np.random.default_rng(3)
    for trial in range(6):
        if trial % 2 == 0:
            s, d, w, loops, part = workloads.regular_bipartite_graph(rng, 7, 3, loop=0.25 * trial)
            n = len(part)
            L = oracle.laplacian(n, s, d, w, loops)
        else:
            s, d, w, loops, part = workloads.random_bipartite_graph(rng, 5, 8)
            n = len(part)
            L = oracle.normalized_laplacian(oracle.laplacian(n, s, d, w, loops))
        c = L[0, 0]
        assert np.allclose(np.diag(L), c, atol=1e-12)
        sigma = np.where(part == 0, 1.0, -1.0)
        lam, U = oracle.gft_basis(L)
        for j in range(n):
            u_hat = sigma * U[:, j]
            assert np.abs(L @ u_hat - (2 * c - lam[j]) * u_hat).max() < 1e-10
        # spectrum symmetric about c
        assert np.abs(np.sort(2 * c - lam) - lam).max() < 1e-10


@pytest.mark.parametrize("n1,n2", [(4, 4), (5, 8), (9, 3), (16, 16), (1, 6), (20, 13)])
def test_normalized_bipartite_right_stage(n1, n2):
    """Theorem 2: normalised Laplacian of a bipartite graph, |S1| != |S2| allowed."""
    rng = np.random.default_rng(100 * n1 + n2)
    s, d, w, loops, part = workloads.random_bipartite_graph(rng, n1, n2, density=0.4)
    n = n1 + n2
    plan = G.Plan(n, s, d, w, loops, host_only=True, normalized=True)
    info = plan.info()
    L = oracle.normalized_laplacian(oracle.laplacian(n, s, d, w, loops))
    _check_basis(L, plan)
    # random weights: no graph symmetry, so the whole graph is one right stage
    assert info["depth"] == 0 and info["n_right_stages"] == 1
    p = min(n1, n2)          # generic: lambda = 1 has multiplicity |n1 - n2| (unpaired)
    assert info["n_right_pairs"] == p
    assert info["n_leaves"] == 2
    assert info["sum_k2"] == n1 * n1 + n2 * n2
    assert info["adds"] == n1 * (n1 - 1) + n2 * (n2 - 1) + 2 * p
    assert info["mults"] == n1 * n1 + n2 * n2
    assert sorted(plan.leaf_sizes()) == sorted([n1, n2])
    # ablation flag: one dense block, same spectrum
    off = G.Plan(n, s, d, w, loops, host_only=True, normalized=True, right_haar=False)
    oi = off.info()
    assert oi["n_right_stages"] == 0 and oi["sum_k2"] == n * n
    assert np.abs(off.eigenvalues() - plan.eigenvalues()).max() < 1e-12


@pytest.mark.parametrize("m,loop", [(3, 0.0), (5, 0.0), (8, 0.5), (16, 0.0), (24, 1.25)])
def test_regular_bipartite_right_stage(m, loop):
    """Theorem 1: weighted k-RBG, unnormalised Laplacian, p = n/2."""
    rng = np.random.default_rng(7 * m)
    s, d, w, loops, part = workloads.regular_bipartite_graph(rng, m, 3, loop=loop)
    n = 2 * m
    plan = G.Plan(n, s, d, w, loops, host_only=True)
    info = plan.info()
    L = oracle.laplacian(n, s, d, w, loops)
    _check_basis(L, plan)
    # a small random union of matchings may still have a graph symmetry (m = 3, 5 here):
    # then Haar units come first and the Theorem-4 leaves lose the constant diagonal
    if m >= 8:
        assert info["depth"] == 0
    if info["depth"] == 0:
        assert info["n_right_stages"] == 1 and info["n_right_pairs"] == m
        assert info["adds"] == 2 * m * (m - 1) + 2 * m


def test_non_constant_diagonal_is_not_split():
    """Unnormalised Laplacian of a non-regular bipartite graph: Lemma 1 does not apply
    (diagonal not constant), so no right stage is formed."""
    rng = np.random.default_rng(5)
    s, d, w, loops, part = workloads.random_bipartite_graph(rng, 5, 7, density=0.5)
    plan = G.Plan(12, s, d, w, loops, host_only=True)
    assert plan.info()["n_right_stages"] == 0
    _check_basis(oracle.laplacian(12, s, d, w, loops), plan)


def test_right_stage_inside_symmetric_graph():
    """Leaves reached after Haar units can be right-split too: the normalised cfg3 (PAPER
    Sec. VI-A grid-like skeleton) -- the basis is still the oracle's."""
    cfg = workloads.config("cfg3")
    plan = G.Plan.from_config(cfg, host_only=True, normalized=True)
    info = plan.info()
    assert info["n_right_stages"] >= 1
    L = oracle.normalized_laplacian(oracle.laplacian(cfg.n, cfg.src, cfg.dst, cfg.w, cfg.self_loops))
    _check_basis(L, plan)
    off = G.Plan.from_config(cfg, host_only=True, normalized=True, right_haar=False)
    assert info["adds"] < off.info()["adds"] and info["sum_k2"] < off.info()["sum_k2"]


def test_canonical_signs_of_right_pairs():
    """Both columns of every pair follow the sign rule (reading A-3) -- the coefficient
    butterfly sign s absorbs the second column's sign."""
    rng = np.random.default_rng(21)
    for trial in range(10):
        s, d, w, loops, part = workloads.random_bipartite_graph(rng, 6, 6 + trial % 3)
        n = len(part)
        plan = G.Plan(n, s, d, w, loops, host_only=True, normalized=True)
        U = plan.basis()
        for j in range(n):
            first = U[np.argmax(np.abs(U[:, j]) > 1e-8), j]
            assert first > 0


def _bipartite_with_twins(seed):
    """Random weighted bipartite graph on 8|8 where S1 nodes 0 and 1 are twins (identical
    neighbours and weights): the transposition (0 1) is its only symmetry (p = 1, Lemma 4);
    with the normalised Laplacian (diagonal 1) a right stage also applies."""
    rng = np.random.default_rng(seed)
    pairs, wts = [], []
    nb0 = [8, 9, 10]
    w0 = rng.uniform(0.5, 2.0, 3)
    for v, x in zip(nb0, w0):
        pairs += [(0, v), (1, v)]
        wts += [x, x]
    for a in range(2, 8):
        for b in range(8, 16):
            if rng.random() < 0.45 or b == 8 + (a % 8):
                pairs.append((a, b))
                wts.append(rng.uniform(0.5, 2.0))
    return workloads._edges(pairs, wts)


def test_right_stage_preferred_over_a_small_left_stage():
    """Reading R-7: with a symmetry of p = 1 the left stage leaves 1 + 15^2 = 226 leaf
    multiplications, the right stage 8^2 + 8^2 = 128 -- the planner takes the right stage,
    and the basis is still the oracle's GFT."""
    s, d, w = _bipartite_with_twins(0)
    L = oracle.normalized_laplacian(oracle.laplacian(16, s, d, w))
    phi, p, _ = G.gft_find_involution(L)
    assert p == 1 and phi[0] == 1
    plan = G.Plan(16, s, d, w, host_only=True, normalized=True)
    info = plan.info()
    assert info["depth"] == 0 and info["n_right_stages"] == 1 and info["sum_k2"] == 128
    _check_basis(L, plan)
    off = G.Plan(16, s, d, w, host_only=True, normalized=True, right_haar=False).info()
    assert off["units_per_level"][0] == 1 and off["sum_k2"] > 128
    # the cycle C64 (2-RBG with p = 32: 2048 = 2048) keeps the left recursion
    cfg = workloads.config("cfg5a")
    assert G.Plan.from_config(cfg, host_only=True).info()["n_right_stages"] == 0
