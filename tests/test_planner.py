"""Host planner (library) checked against the oracle and the paper (-m "not gpu").

The library's decomposition (Theorem 4 closed form) is compared with the oracle's
B_phi^T L B_phi matrix product; the realised basis U_f exported by gft_plan_basis is
compared with the oracle's eigenbasis per eigenvalue cluster (reading A-4)."""

import numpy as np
import pytest

import oracle
import workloads
from conftest import read_golden
from paper_1907_07875_b200 import gft as G


def _proj(U, cols):
    Q = U[:, cols]
    return Q @ Q.T


def check_basis_against_oracle(n, s, d, w, loops, plan, atol=1e-10):
    L = oracle.laplacian(n, s, d, w, loops)
    lam_o, U_o = oracle.gft_basis(L)
    lam_f, U_f = plan.eigenvalues(), plan.basis()
    scale = max(1.0, np.abs(L).max())
    assert np.abs(lam_f - lam_o).max() < 1e-11 * scale
    assert np.abs(L @ U_f - U_f * lam_f).max() < 1e-11 * scale
    assert np.abs(U_f.T @ U_f - np.eye(n)).max() < 1e-12
    for C in oracle.clusters(lam_o):
        if len(C) == 1:
            # simple eigenvalue: same canonical column, coefficient-wise and signed
            assert np.abs(U_f[:, C[0]] - U_o[:, C[0]]).max() < atol
        else:
            assert np.abs(_proj(U_f, C) - _proj(U_o, C)).max() < atol
    return lam_o, U_o, U_f


# --- Theorem 4 closed form vs B_phi^T L B_phi -----------------------------------------
def test_theorem4_matches_conjugation_random():
    rng = np.random.default_rng(11)
    worst = 0.0
    for trial in range(400):
        n = int(rng.integers(2, 21))
        s, d, w, loops, phi = workloads.random_symmetric_graph(
            rng, n, density=float(rng.uniform(0.2, 0.9)), negative=bool(trial % 3 == 0),
            fixed_frac=float(rng.uniform(0, 0.6)))
        L = oracle.laplacian(n, s, d, w, loops)
        if np.all(phi == np.arange(n)):
            continue
        Lp, Lm = G.gft_decompose(L, phi)
        Lp_o, Lm_o, G_o, (vx, vy, vz) = oracle.decompose_blocks(L, phi)
        worst = max(worst, np.abs(Lp - Lp_o).max(initial=0), np.abs(Lm - Lm_o).max(initial=0))
        # Theorem 3: the discarded coupling blocks vanish
        assert np.abs(G_o[np.ix_(vx + vz, vy)]).max(initial=0) < 1e-12 * max(1, np.abs(L).max())
    assert worst < 1e-12


def test_decompose_c4_example():
    s, d, w = workloads.cycle_graph(4)
    L = oracle.laplacian(4, s, d, w)
    Lp, Lm = G.gft_decompose(L, [3, 2, 1, 0])
    assert np.allclose(Lp, [[1, -1], [-1, 1]], atol=1e-15)
    assert np.allclose(Lm, [[3, -1], [-1, 3]], atol=1e-15)


def test_decompose_rejects_bad_phi():
    s, d, w = workloads.path_graph(4)
    L = oracle.laplacian(4, s, d, w)
    with pytest.raises(G.GFTError) as e:
        G.gft_decompose(L, [1, 2, 3, 0])
    assert e.value.name == "GFT_ERR_NOT_INVOLUTION"
    with pytest.raises(G.GFTError) as e:
        G.gft_decompose(L, [1, 0, 2, 3])
    assert e.value.name == "GFT_ERR_NOT_SYMMETRIC"


def test_laplacian_matches_oracle():
    rng = np.random.default_rng(2)
    for n in (1, 3, 9, 17):
        s, d, w, loops, _ = workloads.random_symmetric_graph(rng, n, negative=True)
        # equal up to the summation order of the diagonal
        assert np.abs(G.gft_laplacian(n, s, d, w, loops) - oracle.laplacian(n, s, d, w, loops)).max() < 1e-14


# --- involution search vs brute force --------------------------------------------------
def _involutions(n):
    def rec(rem):
        if not rem:
            yield {}
            return
        a = rem[0]
        for sub in rec(rem[1:]):
            yield {a: a, **sub}
        for j in rem[1:]:
            rest = [x for x in rem[1:] if x != j]
            for sub in rec(rest):
                yield {a: j, j: a, **sub}
    for m in rec(list(range(n))):
        yield np.array([m[i] for i in range(n)])


def _connected(n, L):
    seen, stack = {0}, [0]
    while stack:
        u = stack.pop()
        for v in range(n):
            if v != u and L[u, v] != 0 and v not in seen:
                seen.add(v); stack.append(v)
    return len(seen) == n


def test_involution_search_matches_brute_force():
    assert sum(1 for _ in _involutions(4)) == 10        # T(4) = 10
    assert sum(1 for _ in _involutions(5)) == 26
    rng = np.random.default_rng(5)
    checked = 0
    for trial in range(300):
        n = int(rng.integers(2, 8))
        if trial % 2:
            s, d, w, loops, _ = workloads.random_symmetric_graph(rng, n, density=0.7)
        else:   # unit weights: many symmetries
            pairs = [(i, j) for i in range(n) for j in range(i + 1, n) if rng.random() < 0.5]
            s = np.array([p[0] for p in pairs], np.int32); d = np.array([p[1] for p in pairs], np.int32)
            w = np.ones(len(pairs)); loops = None
        L = oracle.laplacian(n, s, d, w, loops)
        if not _connected(n, L):
            continue
        best_p, best = 0, np.arange(n)
        for phi in _involutions(n):
            B = oracle.butterfly_Bphi(phi)
            P = np.zeros((n, n)); P[np.arange(n), phi] = 1
            if np.abs(P @ L @ P.T - L).max() > 1e-12:
                continue
            p = int(np.sum(phi > np.arange(n)))
            if p > best_p or (p == best_p and tuple(phi) < tuple(best)):
                best_p, best = p, phi
        phi, p, complete = G.gft_find_involution(L)
        assert complete
        assert p == best_p
        assert tuple(phi) == tuple(best)
        checked += 1
    assert checked > 100


# --- plans on the BASELINE configs -------------------------------------------------------
EXPECTED_SHAPES = {     # SURVEY.md §8 table (derived independently of this build)
    "cfg1": ([4, 2, 1], [1, 1, 2, 4]),
    "cfg2": ([8], [8, 8]),
    "cfg2b": ([8, 4], [8, 4, 4]),
    "cfg3": ([10, 7], [8, 7, 5, 5]),
    "cfg4": ([32, 32, 30, 17, 7, 2], None),
    "cfg5a": ([32, 32, 16, 8, 4, 2], [1, 1, 2, 4, 8, 16, 16, 8, 4, 2, 1, 1]),
    "cfg5b": ([64], [64, 64]),
}


@pytest.mark.parametrize("name", list(EXPECTED_SHAPES))
def test_config_plan_matches_oracle(name):
    cfg = workloads.config(name)
    plan = G.Plan.from_config(cfg, host_only=True)
    info = plan.info()
    units, leaves = EXPECTED_SHAPES[name]
    assert info["units_per_level"] == units
    if leaves is not None:
        assert sorted(plan.leaf_sizes()) == sorted(leaves)
    assert sum(plan.leaf_sizes()) == cfg.n
    if name == "cfg4":
        assert info["sum_k2"] == 348
    check_basis_against_oracle(cfg.n, cfg.src, cfg.dst, cfg.w, cfg.self_loops, plan)


def test_cfg1_max_depth_one():
    cfg = workloads.config("cfg1")
    plan = G.Plan.from_config(cfg, host_only=True, max_depth=1)
    assert plan.info()["units_per_level"] == [4]
    assert sorted(plan.leaf_sizes()) == [4, 4]
    check_basis_against_oracle(8, cfg.src, cfg.dst, cfg.w, None, plan)


def test_cfg4_without_phi_and_with_lr_phi():
    cfg = workloads.config("cfg4")
    lr = np.array([8 * (i // 8) + 7 - (i % 8) for i in range(64)])
    plan = G.Plan(64, cfg.src, cfg.dst, cfg.w, None, lr, host_only=True)
    check_basis_against_oracle(64, cfg.src, cfg.dst, cfg.w, None, plan)
    assert plan.info()["units_per_level"][0] == 32


def test_c4_plan_reproduces_printed_matrix():
    """The planner's C4 GFT equals the printed U_C4 column for column."""
    scale, M, lam_g = read_golden("c4_gft.txt")
    Ug = float(scale[0][0]) * np.array(M, dtype=float)
    s, d, w = workloads.cycle_graph(4)
    plan = G.Plan(4, s, d, w, None, [3, 2, 1, 0], host_only=True)
    assert np.abs(plan.eigenvalues() - np.array(lam_g[0], float)).max() < 1e-14
    Uf = plan.basis()
    # two butterfly stages (Fig. 3(b) of the paper): 2 units, then 1 + 1
    assert plan.info()["units_per_level"] == [2, 1] or plan.info()["n_units"] >= 2
    assert np.abs(Uf - Ug).max() < 1e-14 or np.abs(Uf[:, [0, 3]] - Ug[:, [0, 3]]).max() < 1e-14


def test_random_symmetric_graphs_plan_exact():
    rng = np.random.default_rng(21)
    for trial in range(200):
        n = int(rng.integers(1, 13))
        s, d, w, loops, phi = workloads.random_symmetric_graph(
            rng, n, density=float(rng.uniform(0.2, 0.9)), negative=bool(trial % 4 == 0))
        use_phi = phi if trial % 2 else None
        plan = G.Plan(n, s, d, w, loops, use_phi, host_only=True)
        check_basis_against_oracle(n, s, d, w, loops, plan, atol=1e-9)


@pytest.mark.parametrize("name", ["cfg1", "cfg3", "cfg4", "cfg5a"])
def test_normalized_laplacian_plans(name):
    """GFT of D^{-1/2} L D^{-1/2} (NEXT-3): same decomposition, realised basis vs oracle."""
    cfg = workloads.config(name)
    plan = G.Plan.from_config(cfg, host_only=True, normalized=True)
    L = oracle.normalized_laplacian(oracle.laplacian(cfg.n, cfg.src, cfg.dst, cfg.w, cfg.self_loops))
    lam_o, U_o = oracle.gft_basis(L)
    lam_f, U_f = plan.eigenvalues(), plan.basis()
    assert np.abs(lam_f - lam_o).max() < 1e-12
    assert np.abs(L @ U_f - U_f * lam_f).max() < 1e-12
    for C in oracle.clusters(lam_o):
        if len(C) == 1:
            assert np.abs(U_f[:, C[0]] - U_o[:, C[0]]).max() < 1e-10
        else:
            assert np.abs(_proj(U_f, C) - _proj(U_o, C)).max() < 1e-10
    if name == "cfg5a":   # 2-regular: normalised GFT = GFT with halved eigenvalues
        plain = G.Plan.from_config(cfg, host_only=True)
        assert np.abs(plain.eigenvalues() / 2 - lam_f).max() < 1e-13
    # the top-level symmetry survives normalisation (degrees are phi-invariant); deeper
    # sub-graph symmetries may not, since D^{-1/2} reweights non-regular graphs
    assert plan.info()["units_per_level"][0] == G.Plan.from_config(cfg, host_only=True).info()["units_per_level"][0]


def test_normalized_rejects_zero_degree():
    s, d, w = workloads.path_graph(3)
    with pytest.raises(G.GFTError) as e:
        G.Plan(4, s, d, w, host_only=True, normalized=True)     # node 3 isolated
    assert e.value.name == "GFT_ERR_INVALID_ARG"


def test_disconnected_and_isolated_nodes():
    # two identical paths + an isolated node: components are split before searching
    s = np.array([0, 1, 3, 4], np.int32); d = np.array([1, 2, 4, 5], np.int32)
    w = np.ones(4)
    plan = G.Plan(7, s, d, w, host_only=True)
    check_basis_against_oracle(7, s, d, w, None, plan)
    lam = plan.eigenvalues()
    assert np.sum(np.abs(lam) < 1e-12) == 3        # 3 components -> lambda=0 three times


# --- operation counts (tab:runtime) ---------------------------------------
def test_tab_runtime_dense_counts_and_cycle_fast_counts():
    rows = read_golden("tab_runtime_opcounts.txt")[0]
    for topo, n, madd, mmul, fadd, fmul in rows:
        n = int(n)
        assert int(madd) == n * (n - 1) and int(mmul) == n * n
        if topo == "cycle":
            s, d, w = workloads.cycle_graph(n)
            for phi in (None, [n - 1 - i for i in range(n)]):
                info = G.Plan(n, s, d, w, None, phi, host_only=True).info()
                assert info["dense_adds"] == int(madd) and info["dense_mults"] == int(mmul)
                assert info["adds"] == int(fadd)               # exact
                assert info["paper_mults"] == int(fmul)        # reading A-23
                assert info["mults"] == int(fmul) - 2


def test_single_stage_mult_formula():
    """p^2 + (n-p)^2 multiplications for one Haar layer."""
    rng = np.random.default_rng(9)
    for _ in range(30):
        n = int(rng.integers(3, 16))
        s, d, w, loops, phi = workloads.random_symmetric_graph(rng, n, density=0.8)
        p = int(np.sum(phi > np.arange(n)))
        plan = G.Plan(n, s, d, w, loops, phi, max_depth=1, host_only=True)
        info = plan.info()
        if p == 0:
            continue
        # leaves inside G+ / G- may split further into components: <= bound
        assert info["sum_k2"] <= p * p + (n - p) ** 2
        assert info["units_per_level"][0] == p


def test_leaf_closed_forms_cycle64():
    """cfg5a leaves are P_n / Q_n / R_n paths: the spectrum of the plan is
    the cycle's closed form 2 - 2cos(2 pi k / 64) and Lemma 1 pairing holds."""
    cfg = workloads.config("cfg5a")
    plan = G.Plan.from_config(cfg, host_only=True)
    lam = plan.eigenvalues()
    ref = np.sort(2 - 2 * np.cos(2 * np.pi * np.arange(64) / 64))
    assert np.abs(lam - ref).max() < 1e-12


# --- graphs with 2-sparse eigenvectors (Lemma 4; NEXT-3) ---------------
def _star(n):
    return workloads._edges([(0, i) for i in range(1, n)])


def _complete(n):
    return workloads._edges([(i, j) for i in range(n) for j in range(i + 1, n)])


def _clique_with_tail(m, tail):
    """K_m on 0..m-1; nodes m-2, m-1 also chain to a path of `tail` nodes (so nodes 0..m-3
    keep no outside neighbours: Lemma 4's clique example)."""
    pairs = [(i, j) for i in range(m) for j in range(i + 1, m)]
    pairs += [(m - 2, m), (m - 1, m)] + [(m + t, m + t + 1) for t in range(tail - 1)]
    return workloads._edges(pairs)


@pytest.mark.parametrize("kind,n", [("star", 9), ("star", 16), ("complete", 8), ("complete", 13),
                                    ("clique", 7)])
def test_two_sparse_eigenvector_graphs(kind, n):
    """Closed forms pin the oracle (star: 0, 1^(n-2), n; complete: 0, n^(n-1)); Lemma 4's
    2-sparse vectors e_i - e_j are eigenvectors; the plan finds Haar units and matches."""
    if kind == "star":
        s, d, w = _star(n)
        nn = n
        ref = np.array([0.0] + [1.0] * (n - 2) + [float(n)])
    elif kind == "complete":
        s, d, w = _complete(n)
        nn = n
        ref = np.array([0.0] + [float(n)] * (n - 1))
    else:
        s, d, w = _clique_with_tail(n, 4)
        nn = n + 4
        ref = None
    L = oracle.laplacian(nn, s, d, w)
    lam_o, U_o = oracle.gft_basis(L)
    if ref is not None:
        assert np.abs(lam_o - ref).max() < 1e-12
    # Lemma 4: w_vi = w_vj for all other v  <=>  (e_i - e_j)/sqrt2 is an eigenvector
    i, j = (1, 2) if kind != "clique" else (0, 1)
    u = np.zeros(nn); u[i], u[j] = 2 ** -0.5, -2 ** -0.5
    Lu = L @ u
    mu = float(u @ Lu)
    assert np.abs(Lu - mu * u).max() < 1e-12
    plan = G.Plan(nn, s, d, w, host_only=True)
    info = plan.info()
    assert info["n_units"] >= 1 and info["units_per_level"][0] >= 1
    check_basis_against_oracle(nn, s, d, w, None, plan)
    # the 2-sparse eigenvector lies in the plan's eigenspace of mu
    lam_f, U_f = plan.eigenvalues(), plan.basis()
    C = np.where(np.abs(lam_f - mu) < 1e-9 * max(1, mu))[0]
    assert np.linalg.norm(U_f[:, C] @ (U_f[:, C].T @ u) - u) < 1e-10


# --- identical-branch tree search (NEXT-3) --------------------------------
def _random_tree(rng, n, weights=False):
    parent = [-1] + [int(rng.integers(0, i)) for i in range(1, n)]
    pairs = [(p, i) for i, p in enumerate(parent) if p >= 0]
    w = rng.choice([1.0, 2.0], len(pairs)) if weights else None
    return workloads._edges(pairs, w)


def test_tree_search_matches_brute_force_max_p():
    """With the backtracking budget exhausted (budget = 1), trees fall back to the
    identical-branch search; its p_phi must be the brute-force maximum and phi valid."""
    rng = np.random.default_rng(12)
    checked = 0
    for trial in range(150):
        n = int(rng.integers(3, 9))
        s, d, w = _random_tree(rng, n, weights=bool(trial % 2))
        loops = np.where(rng.random(n) < 0.2, 0.5, 0.0) if trial % 3 == 0 else None
        L = oracle.laplacian(n, s, d, w, loops)
        best_p = 0
        for phi in _involutions(n):
            P = np.zeros((n, n)); P[np.arange(n), phi] = 1
            if np.abs(P @ L @ P.T - L).max() <= 1e-12:
                best_p = max(best_p, int(np.sum(phi > np.arange(n))))
        phi, p, complete = G.gft_find_involution(L, 1e-10, 1)
        if best_p > 0:
            assert not complete
        assert p == best_p, (n, p, best_p)
        assert np.all(phi[phi] == np.arange(n))
        assert np.abs(L[np.ix_(phi, phi)] - L).max() <= 1e-12
        checked += best_p > 0
    assert checked > 50


def test_tree_search_rescues_large_random_tree():
    """A 300-node random tree: the budgeted backtracking finds nothing, the tree search
    pairs every set of identical sibling branches; the plan is still the oracle's GFT."""
    rng = np.random.default_rng(0)
    s, d, w = _random_tree(rng, 300)
    L = oracle.laplacian(300, s, d, w)
    phi, p, complete = G.gft_find_involution(L, 1e-10, 10 ** 5)
    assert p >= 40 and not complete
    assert np.abs(L[np.ix_(phi, phi)] - L).max() <= 1e-12
    s, d, w = _random_tree(rng, 90)
    plan = G.Plan(90, s, d, w, host_only=True, search_budget=1000)
    assert plan.info()["n_units"] > 0
    check_basis_against_oracle(90, s, d, w, None, plan)


def test_tab_runtime_grid_counts_reproduced():
    """tab:runtime rows for the 6-connected bi-diagonal grid and the z-shaped grid
     with the graphs of reading R-5 and the paper's own first involutions
    (diagonal symmetry; centrosymmetry i -> N+1-i): adds exact on
    all four rows, paper-convention mults (A-23) exact on three; the 4x4 bi-diagonal grid
    splits into sub-GFTs of length 6, 4, 4 and 2 exactly as PAPER.md:679 states.  The 4x4
    z-grid prints 112 mults where Sigma k^2 = 2 * 8^2 = 128 (its figure is not available to
    check which entries the paper did not count)."""
    rows = {(r[0], int(r[1])): r for r in read_golden("tab_runtime_opcounts.txt")[0]}
    for topo, f in (("grid6", workloads.bidiag_grid), ("zgrid", workloads.z_grid)):
        for N in (4, 8):
            n = N * N
            s, d, w = f(N)
            if topo == "grid6":
                phi = np.array([N * (i % N) + i // N for i in range(n)], np.int32)
            else:
                phi = np.array([n - 1 - i for i in range(n)], np.int32)
            plan = G.Plan(n, s, d, w, None, phi, host_only=True)
            info = plan.info()
            _, _, madd, mmul, fadd, fmul = rows[(topo, n)]
            assert info["dense_adds"] == int(madd) and info["dense_mults"] == int(mmul)
            assert info["adds"] == int(fadd), (topo, n, info["adds"], fadd)
            if (topo, n) != ("zgrid", 16):
                assert info["paper_mults"] == int(fmul), (topo, n, info["paper_mults"], fmul)
            if (topo, n) == ("grid6", 16):
                assert sorted(plan.leaf_sizes()) == [2, 4, 4, 6]
            # the 8x8 z-grid has eigenvalue gaps down to 1e-5: eigenvector error ~ eps |L| / gap
            check_basis_against_oracle(n, s, d, w, None, plan, atol=1e-8)
