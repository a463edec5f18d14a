"""Seeded synthetic workloads shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the method (no Laplacian eigensolve, no butterfly,
no transform).  It only builds the five BASELINE.json graphs as edge lists and draws
the seeded signal batches that both sides consume.  The one piece of linear algebra
here is the GMRF *input* sampler the configs prescribe (precision Q = L + c*I,
sampled with a Cholesky factor), written from the quadratic-form definition of the
precision (eq:lqf) so that it does not share a Laplacian builder
with either the oracle or the library.

Config readings:
  cfg1  path N=8, w=1, phi i<->7-i, 4096 x N(0,1), seed 0
  cfg2  symmetric path N=16, w_i=w_{14-i} ~ U[0.1,1], s_0=s_15=0.5,
        2^22 x sigma_i*N(0,1), sigma from (L+0.01I)^-1, seed 1           (A-15, A-16)
  cfg2b legal two-stage variant of cfg2 (w_0..w_6 palindromic, w_7=0.25)  (A-12)
  cfg3  25-node skeleton (BASELINE topology), arm/leg mirror phi, 2^21 x N(0,1), seed 2
                                                                          
  cfg4  8x8 4-connected grid w=1, no phi (searched), 2^21 GMRF(L+0.05I), seed 3
                                                                          
  cfg5a cycle N=64, phi i<->63-i, 2^20 x N(0,1), seed 4
  cfg5b bipartite 64+64, orbit-drawn edges p=0.1, w~U[0.5,2],
        phi i<->127-i, 2^20 x N(0,1), seed 4                              (A-13)
Beyond the configs (right Haar stages): random connected bipartite graphs
(weights U(0.2, 2), used with the normalised Laplacian) and weighted k-regular bipartite
graphs (unions of random perfect matchings), seeded by the caller.
"""
from __future__ import annotations

import dataclasses
from typing import Optional

import numpy as np

__all__ = ["Config", "CONFIGS", "config", "signals", "path_graph", "cycle_graph",
           "grid_graph", "skeleton25_graph", "random_symmetric_graph", "precision_matrix",
           "random_bipartite_graph", "regular_bipartite_graph", "RIGHT_HAAR_BENCH_CASES", "tab_runtime_graphs",
           "right_haar_bench_graph"]


@dataclasses.dataclass
class Config:
    name: str
    n: int
    src: np.ndarray          # int32 [E]
    dst: np.ndarray          # int32 [E]
    w: np.ndarray            # float64 [E]
    self_loops: Optional[np.ndarray]   # float64 [n] or None
    phi: Optional[np.ndarray]          # int32 [n] or None (auto-detect)
    batch: int
    seed: int
    signal: str              # "normal" | "scaled_gmrf_marginals" | "gmrf"
    gmrf_shift: float = 0.0
    dtypes: tuple = ("f32",)
    max_depth: int = -1
    description: str = ""

    @property
    def edges(self):
        return self.src, self.dst, self.w


def _edges(pairs, weights=None):
    pairs = list(pairs)
    src = np.array([p[0] for p in pairs], dtype=np.int32)
    dst = np.array([p[1] for p in pairs], dtype=np.int32)
    if weights is None:
        w = np.ones(len(pairs), dtype=np.float64)
    else:
        w = np.asarray(weights, dtype=np.float64)
    return src, dst, w


def path_graph(n, weights=None):
    """Line graph 0-1-...-(n-1)."""
    return _edges([(i, i + 1) for i in range(n - 1)], weights)


def cycle_graph(n):
    """Unit-weight cycle."""
    return _edges([(i, (i + 1) % n) for i in range(n)])


def grid_graph(rows, cols):
    """4-connected uniform grid, node = cols*r + c."""
    pairs = []
    for r in range(rows):
        for c in range(cols):
            v = cols * r + c
            if c + 1 < cols:
                pairs.append((v, v + 1))
            if r + 1 < rows:
                pairs.append((v, v + cols))
    return _edges(pairs)


def skeleton25_graph():
    """BASELINE cfg3 skeleton: spine 0-1-2-3-4; arms 5..9, 10..14 chained and attached
    to node 4; legs 15..19, 20..24 chained and attached to node 0 (uniform weights)."""
    pairs = [(i, i + 1) for i in range(4)]
    for base, root in ((5, 4), (10, 4), (15, 0), (20, 0)):
        pairs.append((root, base))
        pairs += [(base + t, base + t + 1) for t in range(4)]
    return _edges(pairs)


def _mirror_phi(n):
    return np.array([n - 1 - i for i in range(n)], dtype=np.int32)


def _cfg2_weights(rng, legal_two_stage=False):
    w = np.zeros(15)
    if legal_two_stage:
        half = rng.uniform(0.1, 1.0, size=4)          # w_0..w_3
        for i in range(4):
            w[i] = half[i]
            w[6 - i] = half[i]                        # palindromic w_0..w_6
        w[7] = 0.25                                   # s^-_8 = 2 w_7 = 0.5 = s^-_15
    else:
        w[:8] = rng.uniform(0.1, 1.0, size=8)         # w_0..w_7
    for i in range(7):
        w[14 - i] = w[i]                              # mirror symmetry w_i = w_{14-i}
    return w


def _cfg5b_edges(rng):
    """Random bipartite 64+64 graph made mirror-symmetric under phi(i)=127-i (A-13):
    each orbit {(a,64+b),(63-b,64+63-a)} of the biadjacency is drawn once."""
    pairs, weights = [], []
    for a in range(64):
        for b in range(64):
            a2, b2 = 63 - b, 63 - a
            if (a2, b2) < (a, b):
                continue                               # orbit already drawn
            present = rng.random() < 0.1
            wt = rng.uniform(0.5, 2.0)
            if not present:
                continue
            pairs.append((a, 64 + b)); weights.append(wt)
            if (a2, b2) != (a, b):
                pairs.append((a2, 64 + b2)); weights.append(wt)
    return _edges(pairs, weights)


def _build(name):
    if name == "cfg1":
        s, d, w = path_graph(8)
        return Config(name, 8, s, d, w, None, _mirror_phi(8), 4096, 0, "normal",
                      description="Line graph N=8, uniform (GFT = DCT-II)")
    if name in ("cfg2", "cfg2b"):
        rng = np.random.default_rng(1)
        wts = _cfg2_weights(rng, legal_two_stage=(name == "cfg2b"))
        s, d, w = path_graph(16, wts)
        loops = np.zeros(16); loops[0] = loops[15] = 0.5
        return Config(name, 16, s, d, w, loops, _mirror_phi(16), 1 << 22, 1,
                      "scaled_gmrf_marginals", gmrf_shift=0.01,
                      description="Symmetric line graph N=16 (video residual GMRF)")
    if name == "cfg3":
        s, d, w = skeleton25_graph()
        phi = np.arange(25, dtype=np.int32)
        for t in range(5):
            phi[5 + t], phi[10 + t] = 10 + t, 5 + t
            phi[15 + t], phi[20 + t] = 20 + t, 15 + t
        return Config(name, 25, s, d, w, None, phi, 1 << 21, 2, "normal",
                      description="25-node human skeleton, left/right mirror")
    if name == "cfg4":
        s, d, w = grid_graph(8, 8)
        return Config(name, 64, s, d, w, None, None, 1 << 21, 3, "gmrf", gmrf_shift=0.05,
                      dtypes=("f32", "f64"), description="8x8 4-connected uniform grid")
    if name == "cfg5a":
        s, d, w = cycle_graph(64)
        return Config(name, 64, s, d, w, None, _mirror_phi(64), 1 << 20, 4, "normal",
                      description="Cycle N=64 (steerable DFT)")
    if name == "cfg5b":
        rng = np.random.default_rng(4)
        s, d, w = _cfg5b_edges(rng)
        return Config(name, 128, s, d, w, None, _mirror_phi(128), 1 << 20, 4, "normal",
                      description="Random bipartite 64+64, mirror pairing imposed")
    raise KeyError(name)


CONFIGS = ("cfg1", "cfg2", "cfg2b", "cfg3", "cfg4", "cfg5a", "cfg5b")


def config(name: str) -> Config:
    return _build(name)


def precision_matrix(cfg: Config, shift: float) -> np.ndarray:
    """Q = shift*I + sum_e w_e (e_i - e_j)(e_i - e_j)^T + diag(s): the GMRF precision
    named by the configs, assembled edge by edge from eq:lqf."""
    n = cfg.n
    q = shift * np.eye(n)
    for i, j, wt in zip(cfg.src, cfg.dst, cfg.w):
        e = np.zeros(n); e[i] = 1.0; e[j] = -1.0
        q += wt * np.outer(e, e)
    if cfg.self_loops is not None:
        q += np.diag(cfg.self_loops)
    return q


def signals(cfg: Config, batch: Optional[int] = None, dtype: str = "f32", seed: Optional[int] = None):
    """Seeded [batch, n] signal matrix (torch CPU tensor), per A-15/A-16."""
    import torch
    b = cfg.batch if batch is None else batch
    sd = cfg.seed if seed is None else seed
    g = torch.Generator(device="cpu").manual_seed(sd)
    tdt = torch.float64 if dtype == "f64" else torch.float32
    if cfg.signal == "normal":
        return torch.randn(b, cfg.n, generator=g, dtype=torch.float32).to(tdt)
    q = precision_matrix(cfg, cfg.gmrf_shift)
    if cfg.signal == "scaled_gmrf_marginals":
        sigma = np.sqrt(np.diag(np.linalg.inv(q)))
        z = torch.randn(b, cfg.n, generator=g, dtype=torch.float32).to(torch.float64)
        return (z * torch.from_numpy(sigma)).to(tdt)
    if cfg.signal == "gmrf":
        c = np.linalg.cholesky(q)                     # Q = C C^T
        cinv = np.linalg.inv(c)                       # x^T = z^T C^{-1}  =>  cov(x) = Q^{-1}
        z = torch.randn(b, cfg.n, generator=g, dtype=torch.float64)
        return (z @ torch.from_numpy(cinv)).to(tdt)
    raise ValueError(cfg.signal)


def signals_device(n: int, batch: int, dtype: str = "f32", seed: int = 0, device: str = "cuda"):
    """Seeded i.i.d. N(0,1) [batch, n] signals drawn ON the device (torch's CUDA generator),
    for inputs too large to draw on the host (the > 4 GiB / > 2^30-row edge-case tests); drawn
    in slabs so no temporary exceeds 1 GiB."""
    import torch
    g = torch.Generator(device=device).manual_seed(seed)
    tdt = torch.float64 if dtype == "f64" else torch.float32
    X = torch.empty(batch, n, dtype=tdt, device=device)
    slab = max(1, (1 << 28) // n)
    for r0 in range(0, batch, slab):
        X[r0:r0 + slab].normal_(generator=g)
    return X


def random_symmetric_graph(rng: np.random.Generator, n: int, density: float = 0.5,
                           loops: bool = True, fixed_frac: float = 0.3, negative: bool = False):
    """Random phi-symmetric graph for property tests: draws a random involution phi and
    weights constant on phi-orbits of node pairs (Definition 2).
    Returns (src, dst, w, self_loops, phi)."""
    perm = rng.permutation(n)
    phi = np.arange(n, dtype=np.int32)
    k = 0
    nfixed = int(round(fixed_frac * n))
    free = list(perm[nfixed:])
    while k + 1 < len(free):
        a, b = free[k], free[k + 1]
        phi[a], phi[b] = b, a
        k += 2
    seen = set()
    pairs, weights = [], []
    for i in range(n):
        for j in range(i + 1, n):
            key = (i, j)
            if key in seen:
                continue
            img = tuple(sorted((int(phi[i]), int(phi[j]))))
            seen.add(key); seen.add(img)
            if img[0] == img[1]:
                continue
            if rng.random() >= density:
                continue
            wt = rng.uniform(-1.0, 2.0) if negative else rng.uniform(0.2, 2.0)
            pairs.append(key); weights.append(wt)
            if img != key:
                pairs.append(img); weights.append(wt)
    s = np.zeros(n)
    if loops:
        for i in range(n):
            if i <= phi[i] and rng.random() < 0.3:
                v = rng.uniform(0.1, 1.0)
                s[i] = v; s[phi[i]] = v
    src, dst, w = _edges(pairs, weights)
    return src, dst, w, s, phi


def random_bipartite_graph(rng: np.random.Generator, n1: int, n2: int, density: float = 0.5,
                           shuffle: bool = True):
    """Random connected weighted bipartite graph on parts S1 (n1 nodes) and S2 (n2 nodes),
    weights U(0.2, 2) (the input of the normalised-Laplacian right Haar stage).
    A spanning tree across the parts keeps it connected for any n1, n2 >= 1.  Node labels are shuffled unless shuffle=False (S1 = 0..n1-1).
    Returns (src, dst, w, self_loops, part) with part[i] in {0, 1}."""
    n = n1 + n2
    lab = rng.permutation(n) if shuffle else np.arange(n)
    A, B = [int(v) for v in lab[:n1]], [int(v) for v in lab[n1:]]
    edges = {}
    # spanning tree: every node of B attaches to a node of A and vice versa
    for j, b in enumerate(B):
        edges[tuple(sorted((A[j % n1], b)))] = rng.uniform(0.2, 2.0)
    for i, a in enumerate(A):
        if i >= n2:
            edges[tuple(sorted((a, B[int(rng.integers(n2))])))] = rng.uniform(0.2, 2.0)
    for i in range(n1 - 1):   # link consecutive A nodes through a shared B node (connectivity)
        b = B[int(rng.integers(n2))]
        edges.setdefault(tuple(sorted((A[i], b))), rng.uniform(0.2, 2.0))
        edges.setdefault(tuple(sorted((A[i + 1], b))), rng.uniform(0.2, 2.0))
    for a in A:
        for b in B:
            if rng.random() < density:
                edges.setdefault(tuple(sorted((a, b))), rng.uniform(0.2, 2.0))
    pairs = sorted(edges)
    src, dst, w = _edges(pairs, [edges[p] for p in pairs])
    part = np.zeros(n, dtype=np.int32)
    part[B] = 1
    return src, dst, w, np.zeros(n), part


def regular_bipartite_graph(rng: np.random.Generator, m: int, n_matchings: int = 3,
                            loop: float = 0.0, shuffle: bool = True):
    """Weighted k-regular bipartite graph (k-RBG) on 2m nodes: the union of
    `n_matchings` random perfect matchings S1 -> S2, matching t with weight U(0.5, 1.5)
    (coinciding edges add up), plus the same self-loop `loop` on every node, so every
    weighted degree is the same.  Returns (src, dst, w, self_loops, part)."""
    n = 2 * m
    lab = rng.permutation(n) if shuffle else np.arange(n)
    A, B = [int(v) for v in lab[:m]], [int(v) for v in lab[m:]]
    edges = {}
    for t in range(n_matchings):
        wt = rng.uniform(0.5, 1.5)
        perm = rng.permutation(m)
        for i in range(m):
            key = tuple(sorted((A[i], B[int(perm[i])])))
            edges[key] = edges.get(key, 0.0) + wt
    pairs = sorted(edges)
    src, dst, w = _edges(pairs, [edges[p] for p in pairs])
    part = np.zeros(n, dtype=np.int32)
    part[B] = 1
    return src, dst, w, np.full(n, float(loop)), part


# Bipartite graphs timed by bench.py's right-Haar table (and AOT-compiled by build.py):
# (label, kind, |S1|, |S2|, dtype); kind "norm" = normalised Laplacian of a random bipartite
# graph (Theorem 2), "reg" = unnormalised Laplacian of a weighted 3-RBG (Theorem 1).
RIGHT_HAAR_BENCH_CASES = [("norm-bipartite 32|32", "norm", 32, 32, "f32"),
                          ("norm-bipartite 64|64", "norm", 64, 64, "f32"),
                          ("3-RBG 64|64", "reg", 64, 64, "f32"),
                          ("norm-bipartite 12|20", "norm", 12, 20, "f64")]


def right_haar_bench_graph(case):
    """(n, src, dst, w, self_loops, normalized) of a RIGHT_HAAR_BENCH_CASES entry."""
    _, kind, a, b, _ = case
    rng = np.random.default_rng(a * 1000 + b)
    if kind == "norm":
        s, d, w, loops, _ = random_bipartite_graph(rng, a, b, density=0.3)
    else:
        s, d, w, loops, _ = regular_bipartite_graph(rng, a, 3, loop=0.0)
    return a + b, s, d, w, loops, kind == "norm"


def bidiag_grid(N=8, a=0.5):
    """Bi-diagonally symmetric 6-connected N x N grid G_b of Sec. VI (
    reading R-5): the 4-connected uniform grid (node = N r + c, w = 1) plus the diagonal edges
    (r, c)-(r+1, c+1) with weight a.  Symmetric about both diagonals."""
    pairs, wts = [], []
    for r in range(N):
        for c in range(N):
            v = N * r + c
            if c + 1 < N:
                pairs.append((v, v + 1)); wts.append(1.0)
            if r + 1 < N:
                pairs.append((v, v + N)); wts.append(1.0)
            if r + 1 < N and c + 1 < N:
                pairs.append((v, v + N + 1)); wts.append(a)
    return _edges(pairs, wts)


def z_grid(N=8, w=2.0):
    """z-shaped N x N grid G_z (reading R-5): horizontal edges
    (r, c)-(r, c+1) with weight 1 and anti-diagonal edges (r, c)-(r+1, c-1) with weight w;
    centrosymmetric under phi(i) = N^2 - 1 - i."""
    pairs, wts = [], []
    for r in range(N):
        for c in range(N):
            v = N * r + c
            if c + 1 < N:
                pairs.append((v, v + 1)); wts.append(1.0)
            if r + 1 < N and c >= 1:
                pairs.append((v, v + N - 1)); wts.append(w)
    return _edges(pairs, wts)


# tab:runtime of Sec. VI-A: the paper's matrix-vs-fast comparison graphs with
# its printed operation counts (matrix adds / mults, fast adds / mults) and C-runtime reduction
# (hardware not stated), re-timed on B200 by bench.py --tables.  The 15-node skeleton exists only
# as a figure and is not rebuilt; the 25-node one is cfg3's topology.
def tab_runtime_graphs():
    diag4 = np.array([4 * (i % 4) + i // 4 for i in range(16)], np.int32)
    diag8 = np.array([8 * (i % 8) + i // 8 for i in range(64)], np.int32)
    return [("Cycle", 12, lambda: cycle_graph(12), None, (132, 144, 44, 30), 52.7),
            ("Cycle", 80, lambda: cycle_graph(80), None, (6320, 6400, 1224, 1078), 79.7),
            ("6-conn. grid", 16, lambda: bidiag_grid(4), diag4, (240, 256, 80, 80), 53.7),
            ("6-conn. grid", 64, lambda: bidiag_grid(8), diag8, (4032, 4096, 1104, 1072), 68.5),
            ("Z-shaped grid", 16, lambda: z_grid(4), np.array([15 - i for i in range(16)], np.int32),
             (240, 256, 128, 112), 41.5),
            ("Z-shaped grid", 64, lambda: z_grid(8), np.array([63 - i for i in range(64)], np.int32),
             (4032, 4096, 2048, 2048), 45.0),
            ("Skeleton", 25, skeleton25_graph, config("cfg3").phi, (600, 625, 272, 282), 47.5)]


# Approximate-GFT comparison of Sec. VI-B, timed by bench.py and
# AOT-compiled by build.py: graph -> (builder, involution used for the Haar stages).
APPROX_BENCH_GRAPHS = {
    "G_b 8x8 bidiag 6-conn a=0.5": (bidiag_grid, np.array([8 * (i % 8) + i // 8 for i in range(64)], np.int32)),
    "G_z 8x8 z-shaped w=2": (z_grid, np.array([63 - i for i in range(64)], np.int32)),
}
APPROX_BENCH_LAYERS = (5, 10, 20, 40)


def approx_bench_plans():
    """[(graph label, variant, plan kwargs)] of the Sec. VI-B comparison: "matrix" is the dense
    kernel of the exact plan, "haar" the exact fast GFT, "approx J" max_depth 0 with J
    layers, "haar+approx J" Haar stages with J-layer leaves."""
    out = []
    for label, (_, phi) in APPROX_BENCH_GRAPHS.items():
        out.append((label, "haar", {"phi": phi}))
        for J in APPROX_BENCH_LAYERS:
            out.append((label, "approx %d" % J, {"phi": None, "max_depth": 0, "approx_layers": J}))
            out.append((label, "haar+approx %d" % J, {"phi": phi, "approx_layers": J}))
    return out


def smoke_bipartite32():
    """The 32|32 bipartite graph of __graft_entry__.smoke() (normalised Laplacian -> a right
    Haar stage with two 32-node tcgen05 leaves); AOT-compiled by build.py."""
    return random_bipartite_graph(np.random.default_rng(7), 32, 32, density=0.3)
