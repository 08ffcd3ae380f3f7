"""One process, several devices: `Pipeline(..., devices=[...])` drives
one part per device through a single handle (pt_config.device_of_stage). Neighbouring parts
exchange activations, gradients and credits by peer stores into each other's comm blocks.

- On a box with one GPU, PT_VIRTUAL_DEVICES=1 maps device ordinals onto the one GPU and splits
  its SMs between the parts (co-resident cooperative kernels). The multi-device handle must then
  equal the single-device pipeline with the same CTAs per stage bit for bit, and the f64 oracle
  within the parity bars.
- With two or more GPUs visible, the `gpu2` tests run the same comparison across real devices
  (peer access over NVLink); they skip on a one-GPU box.
"""

import os

import numpy as np
import pytest

from paper_2210_09147_b200 import engine, model as mdl, streams
from tests.helpers import frob_rel, rel, run_oracle

pytestmark = pytest.mark.gpu


@pytest.fixture
def virtual_devices(monkeypatch):
    monkeypatch.setenv("PT_VIRTUAL_DEVICES", "1")


def _data(widths, T, M, seed=5, loss="mse"):
    st = streams.SmoothStream(widths[0], widths[-1], seed=seed, batch=M)
    xs, ys = st.block(0, T)
    if loss == "softmax_ce":
        ys = np.argmax(ys, axis=-1).astype(np.float64)
    return xs.astype(np.float32), ys.astype(np.float32)


def _compare(widths, counts, devices, T, M=1, opt="sgd", loss="mse", lr=0.02, grid=74, learn=True, seed=4,
             oracle=True):
    m = mdl.mlp(widths, seed=seed, loss=loss)
    xs, ys = _data(widths, T, M, loss=loss)
    x0 = xs[0] if M > 1 else xs[0, 0]
    y0 = ys[0] if M > 1 else ys[0, 0]
    multi = engine.Pipeline(m, counts, opt, lr, x0, y0, devices=devices, learn=learn, timeout_ms=60000)
    assert multi.multi_device
    one = engine.Pipeline(m, counts, opt, lr, x0, y0, grid=grid, learn=learn)
    assert multi.kernel_path == one.kernel_path
    o1, l1, v1 = multi.run(xs, ys)
    o2, l2, v2 = one.run(xs, ys)
    assert np.array_equal(v1, v2)
    assert np.array_equal(o1, o2), float(np.max(np.abs(o1 - o2)))
    assert np.array_equal(l1, l2, equal_nan=True)
    for j in range(one.L):
        (Wa, ba), (Wb, bb) = multi.get_layer(j), one.get_layer(j)
        assert np.array_equal(Wa, Wb) and np.array_equal(ba, bb), j
    if oracle:
        o64, l64, v64, W64, _ = run_oracle(m, counts, xs.astype(np.float64), ys.astype(np.float64), lr,
                                           np.float64, 1, learn, loss, opt)
        assert rel(o1.reshape(o64.shape), o64) <= 1e-4
        if learn:
            W0 = [l.W.astype(np.float64) for l in m.dense_layers]
            for j in range(one.L):
                dW = multi.get_layer(j)[0].astype(np.float64) - W0[j]
                if np.linalg.norm(W64[j] - W0[j]) > 0:
                    assert frob_rel(dW, W64[j] - W0[j]) <= 1e-3, j
    kind = multi.kernel_path
    multi.close()
    one.close()
    return kind


@pytest.mark.parametrize("widths,counts,devices,T,M,opt", [
    ([256, 512, 512, 512, 128], [4, 3], [0, 1], 24, 1, "sgd"),        # panel kernel
    ([64, 96, 96, 96, 96, 32], [4, 2, 3], [0, 1, 2], 30, 1, "sgd"),   # three parts
    ([64, 96, 96, 96, 32], [4, 3], [0, 1], 24, 1, "adam"),            # tick kernel
    ([256, 512, 512, 256, 256], [4, 3], [0, 1], 12, 16, "sgd"),       # tcgen05 tile kernel
])
def test_virtual_devices_match_single_device(virtual_devices, widths, counts, devices, T, M, opt):
    import torch
    grid = torch.cuda.get_device_properties(0).multi_processor_count // len(devices)
    kind = _compare(widths, counts, devices, T, M=M, opt=opt, grid=grid, lr=0.02 if opt == "sgd" else 1e-3)
    assert kind == {1: "panel", 16: "tile"}[M]


def test_virtual_devices_step_api(virtual_devices):
    """Per-sample pipeline_step through a multi-device handle == pipeline_run on one device."""
    import torch
    widths, counts, T = [64, 96, 96, 32], [2, 3], 10
    m = mdl.mlp(widths, seed=2)
    xs, ys = _data(widths, T, 1)
    multi = engine.Pipeline(m, counts, "sgd", 0.05, xs[0, 0], ys[0, 0], devices=["cuda:0", "cuda:1"],
                            timeout_ms=60000)
    one = engine.Pipeline(m, counts, "sgd", 0.05, xs[0, 0], ys[0, 0],
                          grid=torch.cuda.get_device_properties(0).multi_processor_count // 2)
    o, l, v = one.run(xs, ys)
    for t in range(T):
        out = multi.step(xs[t, 0], ys[t, 0])
        assert out.valid == bool(v[t]) and np.array_equal(out.output, o[t, 0])
        if out.valid:
            assert out.loss == float(l[t])
    # device tensors: inputs on stage 1's device, outputs with stage D
    xd, yd = torch.from_numpy(xs).cuda(), torch.from_numpy(ys).cuda()
    o2, l2, _ = multi.run(xd, yd)
    o3, l3, _ = one.run(xs, ys)
    assert np.array_equal(o2.cpu().numpy(), o3) and np.array_equal(l2.cpu().numpy(), l3, equal_nan=True)
    multi.close()
    one.close()


def test_virtual_devices_resident_steps_interleaved(virtual_devices):
    """Per-sample steps on a multi-device handle run as one resident launch per part (all parts
    poll the same mapped request word); runs and weight reads in between stop and restart them.
    The result equals one pt_run on the single-device pipeline, bit for bit."""
    import torch
    widths, counts, T = [48, 80, 80, 80, 10], [2, 2, 3], 24
    m = mdl.mlp(widths, seed=7)
    xs, ys = _data(widths, T, 1, seed=8)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    multi = engine.Pipeline(m, counts, "sgd", 0.05, xs[0, 0], ys[0, 0], devices=[0, 1, 2], timeout_ms=60000)
    one = engine.Pipeline(m, counts, "sgd", 0.05, xs[0, 0], ys[0, 0], grid=sms // 3)
    o_ref, l_ref, _ = one.run(xs, ys)
    outs, t = [], 0
    for seg, kind in ((6, "step"), (5, "run"), (4, "step"), (0, "get"), (9, "step")):
        if kind == "get":
            W, b = multi.get_layer(2)
            multi.set_layer(2, W, b)
        elif kind == "run":
            o, _, _ = multi.run(xs[t:t + seg], ys[t:t + seg])
            outs += list(o[:, 0])
        else:
            for k in range(seg):
                outs.append(multi.step(xs[t + k, 0], ys[t + k, 0]).output)
        t += seg
    assert t == T
    assert np.array_equal(np.array(outs), o_ref[:, 0])
    for j in range(one.L):
        assert all(np.array_equal(u, v) for u, v in zip(multi.get_layer(j), one.get_layer(j)))
    multi.close()
    one.close()


def test_paper_api_devices_list(virtual_devices):
    """partime.pipeline.Pipeline(net, ..., devices=[cuda:0, cuda:1])."""
    import torch
    from paper_2210_09147_b200.partime.pipeline import Pipeline
    torch.manual_seed(0)
    net = torch.nn.Sequential(torch.nn.Linear(32, 64), torch.nn.ReLU(), torch.nn.Linear(64, 64), torch.nn.ReLU(),
                              torch.nn.Linear(64, 8))
    x0, y0 = torch.zeros(32), torch.zeros(8)
    p = Pipeline(net, x0, [2, 3], ["cuda:0", "cuda:1"], True, torch.nn.MSELoss(), y0,
                 (torch.optim.SGD, {"lr": 0.01}))
    assert p._eng.device_of_stage == [0, 1] and p._eng.multi_device
    st = streams.SmoothStream(32, 8, seed=1)
    xs, ys = st.block(0, 12)
    outs = []
    for t in range(12):
        p.forward(torch.from_numpy(xs[t, 0]).float(), torch.from_numpy(ys[t, 0]).float())
        outs.append(p.outputs_buffer.cpu().numpy().copy())
    assert np.all(np.isfinite(outs[-1]))


def test_device_of_stage_errors(virtual_devices):
    """Stages of one device must be contiguous; a device list longer than D is rejected."""
    m = mdl.mlp([16, 16, 16, 16, 8], seed=0)
    x0, y0 = np.zeros(16, np.float32), np.zeros(8, np.float32)
    with pytest.raises(ValueError, match="contiguous"):
        engine.Pipeline(m, [2, 2, 2, 1], "sgd", 0.01, x0, y0, devices=[0, 1, 0, 1])
    with pytest.raises(ValueError, match="at most one device per stage"):
        engine.Pipeline(m, [4, 3], "sgd", 0.01, x0, y0, devices=[0, 1, 2])


# ---- real devices ----------------------------------------------------------------------------

def _ngpu():
    import torch
    return torch.cuda.device_count()


@pytest.mark.gpu2
@pytest.mark.parametrize("widths,counts,M", [([512] * 9, [8, 7], 1), ([512, 1024, 1024, 512, 256], [4, 3], 16)])
def test_two_devices_match_single_device(widths, counts, M):
    """Stage h on GPU h-1 (peer stores over NVLink) == both stages in turn on GPU 0."""
    if _ngpu() < 2:
        pytest.skip("needs two visible GPUs")
    os.environ.pop("PT_VIRTUAL_DEVICES", None)
    _compare(widths, counts, [0, 1], 40 if M == 1 else 12, M=M, grid=0)


@pytest.mark.gpu2
def test_all_devices_c2_layers():
    """C2's 32 x 2048 layers over every visible GPU (up to 8), one stage per GPU."""
    n = min(_ngpu(), 8)
    if n < 2:
        pytest.skip("needs two visible GPUs")
    dense = [32 // n + (1 if i < 32 % n else 0) for i in range(n)]
    counts = [2 * k for k in dense[:-1]] + [2 * dense[-1] - 1]  # dense + relu pairs, linear head
    os.environ.pop("PT_VIRTUAL_DEVICES", None)
    _compare([2048] * 33, counts, list(range(n)), 12, grid=0, lr=1e-3, oracle=False)
