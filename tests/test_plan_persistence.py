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


def _leaf_arrays(data):
    """Offsets of every leaf's pos / slot arrays in a serialised plan (format: serialize.cpp)."""
    import struct
    off = 8 + 4 + 4                                  # magic, version, n
    nops = struct.unpack_from("<Q", data, off)[0]
    off += 8 + 20 * nops
    nleaves = struct.unpack_from("<Q", data, off)[0]
    off += 8
    out = []
    for _ in range(nleaves):
        k = struct.unpack_from("<i", data, off)[0]
        off += 4
        pos_off = off + 8
        off = pos_off + 4 * k
        slot_off = off + 8
        off = slot_off + 4 * k
        out.append((k, pos_off, slot_off))
        for elem in (8, 8, 8):                       # lam, V, M (f64 arrays)
            c = struct.unpack_from("<Q", data, off)[0]
            off += 8 + elem * c
        off += 12                                    # level, right, side
        c = struct.unpack_from("<Q", data, off)[0]   # pair
        off += 8 + 4 * c
        off += 4                                     # approx
        nl = struct.unpack_from("<Q", data, off)[0]
        off += 8
        for _ in range(nl):
            nr = struct.unpack_from("<Q", data, off)[0]
            off += 8 + 24 * nr
        c = struct.unpack_from("<Q", data, off)[0]   # perm
        off += 8 + 4 * c
        c = struct.unpack_from("<Q", data, off)[0]   # scale
        off += 8 + 8 * c
    return out


@pytest.mark.parametrize("which", ["pos", "slot"])
def test_duplicate_leaf_index_rejected(which):
    """Leaf sizes summing to n is not enough: a position read by two leaves (or a coefficient
    slot written twice) is rejected (serialize.cpp cover check)."""
    p = G.Plan.from_config(workloads.config("cfg1"), max_depth=1, host_only=True)
    data = bytearray(p.save())
    (k0, p0, s0), (k1, p1, s1) = _leaf_arrays(bytes(data))[:2]
    assert k0 == k1 == 4
    G.Plan.load(bytes(data), host_only=True)         # the parse above is right: intact loads
    src, dst = (p0, p1) if which == "pos" else (s0, s1)
    data[dst:dst + 4] = data[src:src + 4]            # leaf 1's first index := leaf 0's first
    with pytest.raises(G.GFTError) as e:
        G.Plan.load(bytes(data), host_only=True)
    assert e.value.name == "GFT_ERR_INVALID_ARG"
    assert ("two leaves" if which == "pos" else "written twice") in G.gft_last_error()


def test_tuning_trailer_of_other_kernel_family_is_skipped():
    """A tuned plan loads whatever the load-time flags: a tcgen05-variant record is skipped
    when the plan is regenerated without tensor cores, and an FMA-geometry record when it is
    regenerated with them (capi.cpp deserialize)."""
    cfg = workloads.config("cfg5b")
    p = G.Plan.from_config(cfg, dtypes=("f32",))
    rec = p.tuning("f32", kinds=(0,))[0]
    assert rec[0] == -1 and rec[4] in (0, 1, 2, 3)          # cfg5b forward: a tcgen05 kernel
    alt = 3 if rec[4] != 3 else 0
    p.set_tuning({0: (-1, -1, -1, -1, alt)})
    blob = p.save()
    q = G.Plan.load(blob, dtypes=("f32",))
    assert q.tuning("f32", kinds=(0,))[0][4] == alt
    r = G.Plan.load(blob, dtypes=("f32",), no_tensor_cores=True)
    assert r.tuning("f32", kinds=(0,))[0][4] == -1          # FMA kernel, record skipped
    f = G.Plan.from_config(cfg, dtypes=("f32",), no_tensor_cores=True)
    rf = f.tuning("f32", kinds=(0,))[0]
    f.set_tuning({0: (rf[0], rf[1], rf[2], 150 if rf[3] != 150 else 300, -1)})
    blob = f.save()
    s = G.Plan.load(blob, dtypes=("f32",))  # tensor cores allowed again
    assert s.tuning("f32", kinds=(0,))[0][4] in (0, 1, 2, 3)
