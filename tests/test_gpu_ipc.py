"""Stage handles connected through the IPC export/import path (the one-process-per-GPU
protocol of dist.py: system-scope tagged stores into the neighbour's slots, credits in the
neighbour's memory). Here both handles live in one process on GPU 0 with 74 CTAs each, so
their persistent kernels run concurrently on disjoint SMs: results must equal the
single-handle D=2 pipeline bit for bit.

(The two-process version, one stage per process as in a multi-GPU job, is
tests/test_gpu_ipc_process.py.)"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _sample(xs, M):
    return xs[0] if M > 1 else xs[0, 0]


def _stage_pair(widths, counts, lr, xs, ys, grid=74, M=1):
    from paper_2210_09147_b200 import engine, model as mdl
    m = mdl.mlp(widths, seed=4)
    x0, y0 = _sample(xs, M), _sample(ys, M)
    a = engine.Pipeline(m, counts, "sgd", lr, x0, y0, local_stages=(0, 1), grid=grid, timeout_ms=60000)
    b = engine.Pipeline(m, counts, "sgd", lr, x0, y0, local_stages=(1, 1), grid=grid, timeout_ms=60000)
    a.ipc_import(b.ipc_export(2))
    b.ipc_import(a.ipc_export(1))
    return m, a, b


@pytest.mark.parametrize("widths,counts,T,M,grid", [([32, 64, 64, 64, 16], [4, 3], 12, 1, 74),
                                                    ([256, 512, 512, 512, 128], [4, 3], 40, 1, 74),
                                                    ([256, 512, 512, 256, 256], [4, 3], 12, 16, 64)])
def test_ipc_stage_handles_match_single_handle(widths, counts, T, M, grid):
    """M = 16 with widths % 256 == 0 runs the tcgen05 tile kernel on both handles."""
    import torch
    from paper_2210_09147_b200 import engine, model as mdl, streams
    st = streams.SmoothStream(widths[0], widths[-1], seed=5, batch=M)
    xs, ys = st.block(0, T)
    xs, ys = xs.astype(np.float32), ys.astype(np.float32)
    m, a, b = _stage_pair(widths, counts, 0.05, xs, ys, grid=grid, M=M)
    assert a.kernel_path == b.kernel_path == ("tile" if M == 16 else "panel")
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    a.set_stream(sa)
    b.set_stream(sb)
    xd, yd = torch.from_numpy(xs).cuda(), torch.from_numpy(ys).cuda()
    torch.cuda.synchronize()
    a.run(xd, None, T)
    outs, losses, _ = b.run(None, yd, T)
    a.sync()
    b.sync()
    ref = engine.Pipeline(mdl.mlp(widths, seed=4), counts, "sgd", 0.05, _sample(xs, M), _sample(ys, M),
                          grid=grid)  # same work split (stages in turn on all `grid` CTAs)
    o, l, _ = ref.run(xs, ys)
    assert np.array_equal(outs.cpu().numpy(), o) and np.array_equal(losses.cpu().numpy(), l, equal_nan=True)
    W = [ref.get_layer(j) for j in range(ref.L)]
    mine = [a.get_layer(j) for j in a._local_units()] + [b.get_layer(j) for j in b._local_units()]
    assert all(np.array_equal(x, y) for (x, _), (y, _) in zip(mine, W))
    for p in (a, b, ref):
        p.close()


def test_concurrent_stages_match_two_handles(monkeypatch):
    """The row-owned tick kernel (PT_PANEL=0). One handle with two local stages of equal bytes runs them concurrently, 74 CTAs each
    (DESIGN.md §4.1). Its result must equal two co-resident single-stage handles of 74 CTAs
    exchanging through the IPC path, bit for bit: the same row split, the same protocol."""
    import torch
    from paper_2210_09147_b200 import engine, model as mdl, streams
    monkeypatch.setenv("PT_PANEL", "0")
    widths, counts, T = [256] * 7, [6, 5], 16  # 3 + 3 dense layers of 256 x 256
    st = streams.SmoothStream(widths[0], widths[-1], seed=5)
    xs, ys = st.block(0, T)
    xs, ys = xs.astype(np.float32), ys.astype(np.float32)
    m, a, b = _stage_pair(widths, counts, 0.05, xs, ys, grid=74)
    assert a.kernel_path == b.kernel_path == "tick"
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    a.set_stream(sa)
    b.set_stream(sb)
    xd, yd = torch.from_numpy(xs).cuda(), torch.from_numpy(ys).cuda()
    torch.cuda.synchronize()
    a.run(xd, None, T)
    outs, losses, _ = b.run(None, yd, T)
    a.sync()
    b.sync()
    one = engine.Pipeline(mdl.mlp(widths, seed=4), counts, "sgd", 0.05, xs[0, 0], ys[0, 0], grid=148)
    o, l, _ = one.run(xs, ys)
    assert np.array_equal(outs.cpu().numpy(), o) and np.array_equal(losses.cpu().numpy(), l, equal_nan=True)
    W = [one.get_layer(j) for j in range(one.L)]
    mine = [a.get_layer(j) for j in a._local_units()] + [b.get_layer(j) for j in b._local_units()]
    assert all(np.array_equal(x, y) for (x, _), (y, _) in zip(mine, W))
    for p in (a, b, one):
        p.close()
