"""Per-thread tensor-map cache of the launch path (cuda_rt.cpp): launches that cycle through
more (kernel, buffer, batch) combinations than the cache holds, in place and out of place,
with ragged batches and interleaved kernels, are bit-identical to launches of a fresh plan."""
import pytest

torch = pytest.importorskip("torch")

import workloads  # noqa: E402
from paper_1907_07875_b200 import gft  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg4"])
def test_map_cache_cycles(name):
    cfg = workloads.config(name)
    g = torch.Generator(device="cuda").manual_seed(3)
    cases = []
    for i, rows in enumerate([4096, 4095, 1000, 4096, 37, 2048, 4096]):
        X = torch.randn(rows, cfg.n, generator=g, device="cuda")
        cases.append((X, torch.empty_like(X), i % 3 == 0))
    ref_plan = gft.Plan.from_config(cfg, dtypes=("f32",))
    refs = []
    for X, _, inplace in cases:
        fresh = gft.Plan.from_config(cfg, dtypes=("f32",))   # new kernels: no cache entries
        refs.append((fresh.forward(X), fresh.inverse(X)))
        fresh.close()
    torch.cuda.synchronize()
    for _ in range(3):
        for (X, Y, inplace), (yf, yi) in zip(cases, refs):
            if inplace:
                Z = X.clone()
                ref_plan.forward(Z, Z)
                assert torch.equal(Z, yf)
            ref_plan.forward(X, Y)
            assert torch.equal(Y, yf)
            ref_plan.inverse(X, Y)
            assert torch.equal(Y, yi)
    ref_plan.close()


def test_mixed_cfg5_two_streams_bit_identical():
    """configs[4]'s mixed batch: cfg5a (FMA kernel) and cfg5b (tcgen05 pair kernel) launched
    concurrently on two streams give the same bits as one at a time."""
    ca, cb = workloads.config("cfg5a"), workloads.config("cfg5b")
    pa, pb = gft.Plan.from_config(ca, dtypes=("f32",)), gft.Plan.from_config(cb, dtypes=("f32",))
    g = torch.Generator(device="cuda").manual_seed(4)
    Xa = torch.randn(200_000, ca.n, generator=g, device="cuda")
    Xb = torch.randn(200_000, cb.n, generator=g, device="cuda")
    ra, rb = pa.forward(Xa), pb.forward(Xb)
    torch.cuda.synchronize()
    Ya, Yb = torch.empty_like(ra), torch.empty_like(rb)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(3):
        pa.forward(Xa, Ya, s1)
        pb.forward(Xb, Yb, s2)
    torch.cuda.synchronize()
    assert torch.equal(Ya, ra) and torch.equal(Yb, rb)
    pa.close()
    pb.close()
