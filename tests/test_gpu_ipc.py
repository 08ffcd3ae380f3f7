"""Two processes, one stage each, exchanging activations/gradients through CUDA IPC peer
memory (the one-process-per-GPU path of bench.py/dist.py). Both processes share GPU 0
here, because gpurun hands out one GPU, and their persistent kernels time-slice. Results
must equal the single-process D=2 pipeline, bit for bit."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _worker(rank, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE="2")
    import torch
    import torch.distributed as dist
    from paper_2210_09147_b200 import dist as pdist, model as mdl, streams
    dist.init_process_group("gloo", rank=rank, world_size=2)
    torch.cuda.set_device(0)
    m = mdl.mlp([32, 64, 64, 64, 16], seed=4)
    st = streams.SmoothStream(32, 16, seed=5)
    xs, ys = st.block(0, 12)
    xs, ys = xs.astype(np.float32), ys.astype(np.float32)
    pipe = pdist.build_distributed(m, [4, 3], "sgd", 0.05, xs[0, 0], ys[0, 0], timeout_ms=60000)
    first = pipe.local_first == 0
    outs, losses, valid = pipe.run(torch.from_numpy(xs).cuda() if first else None,
                                   None if first else torch.from_numpy(ys).cuda(), 12)
    pipe.sync()
    res = {"rank": rank, "weights": [pipe.get_layer(j) for j in pipe._local_units()]}
    if not first:
        res["outs"], res["losses"] = outs.cpu().numpy(), losses.cpu().numpy()
    q.put(res)
    dist.barrier()
    pipe.close()
    dist.destroy_process_group()


def test_two_process_ipc_matches_single_process():
    import torch.multiprocessing as mp
    from paper_2210_09147_b200 import engine, model as mdl, streams
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = {}
    for _ in procs:
        r = q.get(timeout=300)
        got[r["rank"]] = r
    for p in procs:
        p.join(timeout=120)
    m = mdl.mlp([32, 64, 64, 64, 16], seed=4)
    st = streams.SmoothStream(32, 16, seed=5)
    xs, ys = st.block(0, 12)
    ref = engine.Pipeline(m, [4, 3], "sgd", 0.05, xs[0, 0], ys[0, 0])
    o, l, v = ref.run(xs.astype(np.float32), ys.astype(np.float32))
    assert np.array_equal(got[1]["outs"], o) and np.array_equal(got[1]["losses"], l, equal_nan=True)
    W = [ref.get_layer(j) for j in range(ref.L)]
    assert all(np.array_equal(a, b) for (a, _), (b, _) in zip(got[0]["weights"] + got[1]["weights"], W))
