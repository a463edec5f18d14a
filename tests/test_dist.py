"""Multi-process host logic of the batch-sharded path (gloo, world_size 2, CPU)."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1907_07875_b200 import dist as D


def test_shard_rows_cover_exactly():
    for batch in (0, 1, 7, 4096, 2 ** 21 + 3):
        for world in (1, 2, 3, 8):
            spans = [D.shard_rows(batch, r, world) for r in range(world)]
            assert spans[0][0] == 0
            for (s0, c0), (s1, c1) in zip(spans, spans[1:]):
                assert s0 + c0 == s1
            assert spans[-1][0] + spans[-1][1] == batch
            assert max(c for _, c in spans) - min(c for _, c in spans) <= 1
    with pytest.raises(ValueError):
        D.shard_rows(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import workloads
    from paper_1907_07875_b200 import gft as G
    ws, rk, _ = D.dist_env()
    assert (ws, rk) == (world, rank)
    # every rank builds the same plan (deterministic planner / codegen)
    cfg = workloads.config("cfg3")
    plan = G.Plan.from_config(cfg, host_only=False, dtypes=("f32",))
    name = plan.kernel_name(0, "f32")
    basis = plan.basis()
    names = [None] * world
    dist.all_gather_object(names, name)
    bases = [None] * world
    dist.all_gather_object(bases, basis.tobytes())
    # per-rank timing reduced with MAX
    t = D.max_over_ranks(1.0 + rank)
    start, count = D.shard_rows(1000, rank, world)
    counts = [None] * world
    dist.all_gather_object(counts, (start, count))
    D.barrier()
    out[rank] = (names, bases[0] == bases[-1], t, counts)
    dist.destroy_process_group()


def test_two_ranks_gloo():
    world, port = 2, _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    for r in range(world):
        names, same_basis, t, counts = out[r]
        assert len(set(names)) == 1          # identical generated kernels on every rank
        assert same_basis
        assert t == 2.0                      # MAX over ranks
        assert sum(c for _, c in counts) == 1000
