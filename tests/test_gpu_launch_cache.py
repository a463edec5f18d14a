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
