"""Plan persistence (gft_plan_serialize / gft_plan_deserialize): a saved plan reloads with
the same basis, eigenvalues, statistics and generated kernels (names = source hashes), for
left Haar stages, right Haar stages, approximate leaves and the normalised Laplacian; and
malformed bytes are rejected with GFT_ERR_INVALID_ARG, never a crash."""
import numpy as np
import pytest

import workloads
from paper_1907_07875_b200 import gft as G


def _plans():
    out = []
    for name in ("cfg1", "cfg3", "cfg4", "cfg5b"):
        out.append((name, G.Plan.from_config(workloads.config(name), dtypes=("f32", "f64"))))
    s, d, w, loops, _ = workloads.random_bipartite_graph(np.random.default_rng(1), 12, 20, density=0.3)
    out.append(("right_haar", G.Plan(32, s, d, w, loops, normalized=True)))
    s, d, w = workloads.bidiag_grid()
    out.append(("approx", G.Plan(64, s, d, w, approx_layers=15)))
    return out


@pytest.mark.parametrize("idx", range(6))
def test_round_trip(idx):
    name, p = _plans()[idx]
    data = p.save()
    q = G.Plan.load(data)
    assert q.info() == p.info(), name
    assert np.array_equal(q.basis(), p.basis()) and np.array_equal(q.eigenvalues(), p.eigenvalues())
    assert q.leaf_sizes() == p.leaf_sizes()
    for dt in ("f32", "f64"):
        for k in range(4):
            assert q.kernel_name(k, dt) == p.kernel_name(k, dt)
    assert q.save() == data                        # stable re-serialisation


def test_host_only_load_and_dtype_subset():
    p = G.Plan.from_config(workloads.config("cfg2"), host_only=True)
    q = G.Plan.load(p.save(), host_only=True)
    assert np.array_equal(q.basis(), p.basis())
    r = G.Plan.load(p.save(), dtypes=("f32",))
    assert r.kernel_name(0, "f32").startswith("gft_fwd_f32_n16_")
    with pytest.raises(G.GFTError):
        r.kernel_name(0, "f64")


def test_malformed_bytes_rejected():
    data = bytearray(G.Plan.from_config(workloads.config("cfg3"), host_only=True).save())
    for bad in (b"", b"GFTPLAN1", bytes(data[:-1]), bytes(data) + b"\x00",
                b"NOTAPLAN" + bytes(data[8:])):
        with pytest.raises(G.GFTError) as e:
            G.Plan.load(bad, host_only=True)
        assert e.value.name == "GFT_ERR_INVALID_ARG"
    rng = np.random.default_rng(0)
    for _ in range(200):                            # random byte flips: error or a valid plan
        mutated = bytearray(data)
        for i in rng.integers(12, len(data), size=3):
            mutated[i] ^= int(rng.integers(1, 256))
        try:
            G.Plan.load(bytes(mutated), host_only=True)
        except G.GFTError as e:
            assert e.name in ("GFT_ERR_INVALID_ARG", "GFT_ERR_UNSUPPORTED")


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["cfg2", "cfg4", "cfg5b"])
def test_loaded_plan_bit_identical_on_gpu(name):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    p = G.Plan.from_config(workloads.config(name), dtypes=("f32",))
    q = G.Plan.load(p.save(), dtypes=("f32",))
    n = p.n
    g = torch.Generator(device="cuda").manual_seed(3)
    X = torch.randn(4099, n, device="cuda", generator=g)
    Yp, Yq = p.forward(X), q.forward(X)
    assert torch.equal(Yp, Yq)
    assert torch.equal(p.inverse(Yp), q.inverse(Yq))
