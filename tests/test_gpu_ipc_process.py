"""Two processes, one stage each, exchanging activations and gradients through CUDA IPC
peer memory: the one-process-per-GPU path of bench.py / dist.py (build_distributed,
exchange_ipc over a gloo group). gpurun hands out one GPU, so both processes share GPU 0
and the driver time-slices their persistent kernels. Results must still equal the
single-process D=2 pipeline bit for bit: the batch-1 and micro-batch tick kernel and the
tcgen05 tile kernel. (Time-sliced runs are bitwise equal to solo runs once legacy-stream
work is ordered before the handle's stream; tools/timeslice_probe.py.)"""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

# (widths, counts, ticks, batch)
CASES = {"panel": ([32, 64, 64, 64, 16], [4, 3], 12, 1),
         "panel_wide": ([256, 512, 512, 512, 128], [4, 3], 24, 1),
         "tick": ([32, 64, 64, 64, 16], [4, 3], 12, 1),
         "tick_microbatch": ([64, 96, 96, 96, 32], [4, 3], 16, 4),
         "tile": ([256, 512, 512, 256, 256], [4, 3], 12, 16)}


def _data(case):
    from paper_2210_09147_b200 import streams
    widths, counts, T, M = CASES[case.replace("_2gpu", "")]
    st = streams.SmoothStream(widths[0], widths[-1], seed=5, batch=M)
    xs, ys = st.block(0, T)
    return widths, counts, T, M, xs.astype(np.float32), ys.astype(np.float32)


def _sample(a, M):
    return a[0] if M > 1 else a[0, 0]


def _worker(rank, port, q, case):
    if case.startswith("tick"):
        os.environ["PT_PANEL"] = "0"  # the row-owned tick kernel
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE="2")
    import torch
    import torch.distributed as dist
    from paper_2210_09147_b200 import dist as pdist, model as mdl
    dist.init_process_group("gloo", rank=rank, world_size=2)
    # "_2gpu" cases: one GPU per process (NVLink peer stores through CUDA IPC), else both on GPU 0
    torch.cuda.set_device(rank if case.endswith("_2gpu") else 0)
    widths, counts, T, M, xs, ys = _data(case)
    pipe = pdist.build_distributed(mdl.mlp(widths, seed=4), counts, "sgd", 0.05, _sample(xs, M), _sample(ys, M),
                                   timeout_ms=60000)
    first = pipe.local_first == 0
    outs, losses, valid = pipe.run(torch.from_numpy(xs).cuda() if first else None,
                                   None if first else torch.from_numpy(ys).cuda(), T)
    pipe.sync()
    res = {"rank": rank, "path": pipe.kernel_path, "weights": [pipe.get_layer(j) for j in pipe._local_units()]}
    if not first:
        res["outs"], res["losses"] = outs.cpu().numpy(), losses.cpu().numpy()
    q.put(res)
    dist.barrier()
    pipe.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("case", list(CASES) + [pytest.param("panel_2gpu", marks=pytest.mark.gpu2),
                                                pytest.param("tile_2gpu", marks=pytest.mark.gpu2)])
def test_two_process_ipc_matches_single_process(case):
    import torch
    import torch.multiprocessing as mp
    from paper_2210_09147_b200 import engine, model as mdl
    if case.endswith("_2gpu") and torch.cuda.device_count() < 2:
        pytest.skip("needs two visible GPUs")
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, port, q, case)) for r in range(2)]
    for p in procs:
        p.start()
    got = {}
    for _ in procs:
        r = q.get(timeout=150)
        got[r["rank"]] = r
    for p in procs:
        p.join(timeout=120)
    widths, counts, T, M, xs, ys = _data(case)
    assert got[0]["path"] == got[1]["path"] == case.split("_")[0]
    # the single-process reference runs its two stages in turn on the whole grid, like each
    # process does with its one stage
    os.environ["PT_CONC"] = "0"
    if case.startswith("tick"):
        os.environ["PT_PANEL"] = "0"
    try:
        ref = engine.Pipeline(mdl.mlp(widths, seed=4), counts, "sgd", 0.05, _sample(xs, M), _sample(ys, M))
    finally:
        os.environ.pop("PT_CONC", None)
        os.environ.pop("PT_PANEL", None)
    o, l, v = ref.run(xs, ys)
    assert np.array_equal(got[1]["outs"], o) and np.array_equal(got[1]["losses"], l, equal_nan=True)
    W = [ref.get_layer(j) for j in range(ref.L)]
    assert all(np.array_equal(a, b) for (a, _), (b, _) in zip(got[0]["weights"] + got[1]["weights"], W))
    ref.close()
