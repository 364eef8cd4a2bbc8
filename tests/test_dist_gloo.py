"""Multi-rank host logic on CPU (gloo, world_size 2): x-mode slab partition, the all-reduce(max)
callback the plans use, and the modal-slab gather + assembly of the output path."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2007_13125_b200 import dist as pdist
from paper_2007_13125_b200 import pint


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, mx, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        qb, qe = pint.partition(mx, rank, world)
        # all-reduce(max) callback: every rank must see the max of the per-rank updates
        red = pdist.make_allreduce_max()
        got = red(float(10 * rank + 3.5))
        # modal slab gather: rank's slab of a known global array
        rng = np.random.default_rng(0)
        full = rng.standard_normal((3, 5, mx)) + 1j * rng.standard_normal((3, 5, mx))
        g = pdist.gather_modal(np.ascontiguousarray(full[:, :, qb:qe]), mx)
        q.put((rank, qb, qe, got, bool(np.array_equal(g, full))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mx", [1023, 511, 7])
def test_two_rank_partition_allreduce_gather(mx):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mx, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    bounds = [(r[1], r[2]) for r in res]
    assert bounds[0][0] == 0 and bounds[-1][1] == mx and bounds[0][1] == bounds[1][0]
    assert abs((bounds[0][1] - bounds[0][0]) - (bounds[1][1] - bounds[1][0])) <= 1
    assert all(r[3] == 13.5 for r in res)          # max(3.5, 13.5)
    assert all(r[4] for r in res)


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_partition_tiles_modes(world):
    mx = 1023
    b = [pint.partition(mx, r, world) for r in range(world)]
    assert b[0][0] == 0 and b[-1][1] == mx
    assert all(b[i][1] == b[i + 1][0] for i in range(world - 1))
    sizes = [e - s for s, e in b]
    assert max(sizes) - min(sizes) <= 1


def test_partition_rejects():
    with pytest.raises(pint.PintError):
        pint.partition(4, 0, 5)
    with pytest.raises(pint.PintError):
        pint.partition(4, 2, 2)


def test_assemble_modal_checks():
    s = [np.zeros((1, 2, 3)), np.zeros((1, 2, 2))]
    assert pdist.assemble_modal(s, [(0, 3), (3, 5)], 5).shape == (1, 2, 5)
    with pytest.raises(ValueError):
        pdist.assemble_modal(s, [(0, 3), (2, 4)], 5)
