"""Multi-process host logic on CPU (gloo, world_size 2): stage assignment and the CUDA-IPC
handle exchange between neighbouring ranks (paper_2210_09147_b200.dist)."""

import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2210_09147_b200 import dist as pdist


def test_stage_range():
    assert [pdist.stage_range(r, 2, 8) for r in range(2)] == [(0, 4), (4, 4)]
    assert [pdist.stage_range(r, 3, 8) for r in range(3)] == [(0, 3), (3, 3), (6, 2)]
    assert [pdist.stage_range(r, 8, 8) for r in range(8)] == [(r, 1) for r in range(8)]
    with pytest.raises(ValueError):
        pdist.stage_range(0, 4, 2)


class FakePipe:
    def __init__(self, rank, world, D):
        self.D = D
        self.local_first, self.local_count = pdist.stage_range(rank, world, D)
        self.imported = []

    def ipc_export(self, h):
        return f"blob-of-stage-{h}".encode()

    def ipc_import(self, blob):
        self.imported.append(blob.decode())


def _worker(rank, world, port, D, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    p = FakePipe(rank, world, D)
    want = pdist.exchange_ipc(p)
    # max-over-ranks timing, as bench.py reports it
    import torch
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    q.put((rank, want, p.imported, float(t[0])))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,D", [(2, 2), (2, 4)])
def test_ipc_exchange_gloo(world, D):
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, D, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in procs:
        r, want, imported, tmax = q.get(timeout=120)
        res[r] = (want, imported, tmax)
    for p in procs:
        p.join(timeout=60)
    per = D // world
    # rank 0 owns stages 1..per and imports the downstream stage per+1; rank 1 the upstream one
    assert res[0][0] == [per + 1] and res[0][1] == [f"blob-of-stage-{per + 1}"]
    assert res[1][0] == [per] and res[1][1] == [f"blob-of-stage-{per}"]
    assert res[0][2] == res[1][2] == float(world)
