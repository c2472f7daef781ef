"""Multi-process (N>1) host logic on CPU with the gloo backend, world size 2:
the batch shards are disjoint and cover the sweep, every rank builds the same
tile pattern (so one plan serves all its matrices), and the MAX-over-ranks
time reduction used by bench.py picks the slowest rank."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2504_19171_b200.shard import batch_seeds, max_over_ranks, shard_range


def test_shard_range_partition():
    for count in (0, 1, 7, 64, 65):
        for world in (1, 2, 3, 8):
            got = [shard_range(count, r, world) for r in range(world)]
            assert got[0][0] == 0 and got[-1][1] == count
            assert all(a[1] == b[0] for a, b in zip(got, got[1:]))
            sizes = [e - s for s, e in got]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2504_19171_b200 as tib

    seeds = batch_seeds(1000, 64, rank, world)
    # every member of the sweep shares one tile pattern -> one device plan per rank
    pats = {tuple(tib.factor_pattern(tib.generate(2000, 50, 5, 1.0, seed=s, tile_size=128))) for s in seeds[:3]}
    slow = max_over_ranks(1.5 if rank == 1 else 0.5, dist)
    q.put((rank, seeds, len(pats), slow))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_two_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    seeds = out[0][1] + out[1][1]
    assert seeds == list(range(1000, 1064))
    assert all(o[2] == 1 for o in out)
    assert all(o[3] == 1.5 for o in out)
