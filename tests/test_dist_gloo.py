"""World-size-2 gloo run of the batch-axis sharding and the timing reductions
bench.py uses under torchrun (CPU; the GPU path differs only in the device)."""

import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_1409_5254_b200 import dist as tdist


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ws, r, lr = tdist.env()
    ids = tdist.problem_ids(r, ws, 64)
    elapsed = 1.0 + r          # rank 1 is slower
    dofs = float(len(ids) * 10)
    t, w = tdist.reduce_time_and_work(elapsed, dofs)
    out[rank] = (ids[0], ids[-1], t, w)
    dist.destroy_process_group()


def test_two_rank_sharding_and_reduction():
    world = 2
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    assert res[0][:2] == (0, 63) and res[1][:2] == (64, 127)   # disjoint problem ids
    for r in range(world):
        assert res[r][2] == 2.0        # max over ranks
        assert res[r][3] == 1280.0     # total work


def test_single_process_identity():
    assert tdist.reduce_time_and_work(1.5, 7.0) == (1.5, 7.0)
    assert tdist.problem_ids(0, 1, 3) == [0, 1, 2]
    with pytest.raises(ValueError):
        tdist.problem_ids(2, 2, 3)
