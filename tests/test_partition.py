"""Partitioned single-matrix path (paper_2504_19171_b200/partition.py,
SURVEY.md 8(e)): tile-column interiors, separators and the arrow-tip Schur
complement reduced over the process group, checked against the oracle on
Sigma (the matrix's own tile pattern), diag(Sigma) and logdet.

CPU: the orchestration on the dense numpy engine (tests/partition_sim.py,
the prototype), one process and a gloo world of 2.  GPU: the device engine
(factorize, border tile replacement, selected inversion of the modified
factor, the reduced system) with every part in one process."""
import os
import socket

import numpy as np
import pytest

from paper_2504_19171_b200 import partition as P
from partition_sim import NumpyEngine

TOL = 1e-10

CASES = [
    # n, w, t, b: one-tile arrow, two-tile arrow (the arrow straddles a tile row), wider band
    (1500, 60, 12, 32),
    (1000, 60, 12, 32),
    (2600, 130, 20, 32),
]


def check(tib, orc, n, w, t, b, seed, sigma, diag, ld):
    ref = orc.selected_inverse_generated(n, w, t, 1.0, seed, b, "pattern")
    assert abs(ld - ref["logdet"]) <= TOL * abs(ref["logdet"])
    assert np.max(np.abs(diag - ref["diag"]) / np.abs(ref["diag"])) <= TOL
    scale = np.abs(ref["payload"]).max()
    assert set(sigma) == set(map(tuple, ref["tiles"]))
    for k, (i, j) in enumerate(ref["tiles"]):
        hi, hj = min(b, n - i * b), min(b, n - j * b)
        assert np.abs(sigma[(i, j)][:hi, :hj] - ref["payload"][k][:hi, :hj]).max() <= TOL * scale


def test_partition_layout():
    part = P.BandArrowPartition(391, 4, 8)
    assert len(part.interiors) == 8 and all(len(s) == 4 for s in part.seps)
    cols = sorted(c for x in part.interiors + part.seps for c in x)
    assert cols == list(range(390)) and part.arrow == [390]
    # the first part (no left separator, no fill-in) carries the most columns
    assert len(part.interiors[0]) > 2 * len(part.interiors[1])
    for p in range(8):
        order = part.local_order(p)
        assert order[-1] == 390 and len(set(order)) == len(order)
    with pytest.raises(ValueError):
        P.BandArrowPartition(12, 4, 3)


@pytest.mark.parametrize("n,w,t,b", CASES)
@pytest.mark.parametrize("parts", [1, 2, 3])
def test_prototype_matches_oracle(tib, orc, n, w, t, b, parts):
    seed = 5
    m = tib.generate(n, w, t, 1.0, seed=seed, tile_size=b)
    res, red, ld, part, A = P.selected_inverse_partitioned(m, parts, engine=NumpyEngine())
    sigma, diag = P.assemble(A, part, res, red)
    check(tib, orc, n, w, t, b, seed, sigma, diag, ld)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, here)
    sys.path.insert(0, os.path.dirname(here))
    import torch.distributed as dist

    import paper_2504_19171_b200 as tib
    from paper_2504_19171_b200 import partition as PP
    from partition_sim import NumpyEngine as NE

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    m = tib.generate(1500, 60, 12, 1.0, seed=5, tile_size=32)
    res, red, ld, part, A = PP.selected_inverse_partitioned(m, world, rank, world, PP.dist_allreduce(dist),
                                                            engine=NE())
    got = [None] * world
    dist.all_gather_object(got, res)
    if rank == 0:
        sigma, diag = PP.assemble(A, part, [r for rs in got for r in rs], red)
        q.put((sigma, diag, ld))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_two_ranks_prototype(tib, orc):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    sigma, diag, ld = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    check(tib, orc, 1500, 60, 12, 32, 5, sigma, diag, ld)


@pytest.mark.gpu
@pytest.mark.parametrize("n,w,t,b,parts", [(6000, 300, 40, 64, 2), (6000, 300, 40, 64, 3), (9000, 500, 60, 128, 2),
                                           (4100, 200, 70, 64, 3)])
def test_device_partitioned_matches_oracle(tib, orc, n, w, t, b, parts):
    seed = 11
    m = tib.generate(n, w, t, 1.0, seed=seed, tile_size=b)
    res, red, ld, part, A = P.selected_inverse_partitioned(m, parts, device=0)
    sigma, diag = P.assemble(A, part, res, red)
    check(tib, orc, n, w, t, b, seed, sigma, diag, ld)
