"""Maximum-size edge cases on the GPU: buffers larger than 4 GiB (byte offsets beyond 32 bits
in every data path: TMA tensor boxes, the packed 128-B view, 1-D bulk copies of odd pitches,
the tcgen05 kernels, fp64) and a batch larger than 2^30 rows (the library splits it into
launches of at most 2^30 rows: TMA coordinates are int32).  Every row is checked for Parseval
on the device; rows around each boundary (first / last rows, the 4 GiB byte offset, the
2^30-row launch split) plus random rows are compared with the CPU oracle."""
import numpy as np
import pytest

import oracle
import workloads
from paper_1907_07875_b200 import gft as G

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = {"f32": 1e-5, "f64": 1e-12}


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.init()


def _graph(name):
    if name == "path2":   # one edge: a single Haar unit, two 1 x 1 leaves
        return 2, np.array([0], np.int32), np.array([1], np.int32), np.array([1.0]), None, None
    cfg = workloads.config(name)
    return cfg.n, cfg.src, cfg.dst, cfg.w, cfg.self_loops, cfg.phi


def _sample_rows(batch, row_bytes, rng):
    marks = [0, batch - 1, (1 << 32) // row_bytes, (1 << 33) // row_bytes, 1 << 30]
    rows = [rng.integers(0, batch, 1500)]
    for m in marks:
        rows.append(np.arange(max(0, m - 300), min(batch, m + 300)))
    return np.unique(np.concatenate(rows))


def _parseval_all_rows(X, Y, tol):
    worst = 0.0
    slab = max(1, (1 << 26) // X.shape[1])
    for r0 in range(0, X.shape[0], slab):
        nx = torch.linalg.vector_norm(X[r0:r0 + slab].double(), dim=1)
        ny = torch.linalg.vector_norm(Y[r0:r0 + slab].double(), dim=1)
        worst = max(worst, float((ny / nx - 1).abs().max()))
    assert worst < 10 * tol, worst


CASES = [("path2", "f32", (1 << 30) + 4099, False),   # > 2^30 rows: two launches; packed view; 8.6 GB per buffer
         ("cfg1", "f32", (1 << 27) + 3, True),        # packed 128-B view, 4.3 GB, in place
         ("cfg3", "f32", (1 << 26) + 37, False),      # odd pitch: 1-D bulk copies, 6.7 GB per buffer
         ("cfg5a", "f32", (1 << 24) + 77, True),      # TMA tensor boxes, 4.3 GB, in place
         ("cfg5b", "f32", (1 << 23) + 129, False),    # tcgen05 IO-split kernel, 4.3 GB per buffer
         ("cfg4", "f64", (1 << 23) + 5, False)]       # fp64, 4.3 GB per buffer


@pytest.mark.parametrize("name,dtype,batch,in_place", CASES)
def test_large_buffers_vs_oracle(name, dtype, batch, in_place):
    n, src, dst, w, loops, phi = _graph(name)
    elem = 8 if dtype == "f64" else 4
    need = 2 * batch * n * elem + (3 << 30)
    free, _ = torch.cuda.mem_get_info()
    if free < need:
        pytest.skip("needs %.1f GB of free device memory" % (need / 1e9))
    max_depth = -1 if name == "path2" else workloads.config(name).max_depth
    plan = G.Plan(n, src, dst, w, self_loops=loops, phi=phi, dtypes=(dtype,), max_depth=max_depth)
    L = oracle.laplacian(n, src, dst, w, loops)
    lam_o, U_o = oracle.gft_basis(L)
    U_f = plan.basis()
    tol = TOL[dtype]
    X = workloads.signals_device(n, batch, dtype, seed=11)
    assert X.numel() * elem > (1 << 32)
    rows = _sample_rows(batch, n * elem, np.random.default_rng(5))
    idx = torch.from_numpy(rows).cuda()
    Xs = X[idx].cpu().numpy()
    if in_place:
        Y = X.clone()
        plan.forward(Y, Y)
    else:
        Y = plan.forward(X)
    torch.cuda.synchronize()
    _parseval_all_rows(X, Y, tol)
    Ys = Y[idx].cpu().numpy()
    Y_o = oracle.forward(Xs, U_o)
    R = oracle.cluster_rotation(U_o, U_f, lam_o)
    assert oracle.aligned_error(Ys, Y_o, R).max() <= tol
    assert oracle.energy_error(Ys, Y_o, lam_o).max() <= tol
    # inverse over the same buffers gives the sampled rows back
    Xr = plan.inverse(Y, Y)
    torch.cuda.synchronize()
    assert oracle.relative_error(Xr[idx].cpu().numpy(), Xs).max() <= 2 * tol
    del X, Y, Xr
    torch.cuda.empty_cache()
    plan.close()
