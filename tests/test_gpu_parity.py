"""GPU parity: the B200 engine vs the CPU oracle (f64) on the same seeded stream.

Tolerances (fp32 GPU vs f64 oracle). The f32 run of the oracle
calibrates each bar: the GPU error must stay within 4x the oracle's own f32
error, plus a floor of 1e-6 of the signal scale. Stated absolute ceilings:
outputs and losses rel <= 1e-4 per tick; final weights and
delta-W = W_N - W_0 rel-Frobenius <= 1e-3.
"""

import numpy as np
import pytest

from paper_2210_09147_b200 import engine, model as mdl, streams
from tests.helpers import frob_rel, rel, run_oracle

pytestmark = pytest.mark.gpu


def _case(widths, counts, T, lr, act="relu", seed=0, act_delay=1, learn=True, M=1, grid=0):
    m = mdl.mlp(widths, act=act, seed=seed)
    st = streams.SmoothStream(widths[0], widths[-1], seed=seed + 1, batch=M)
    xs, ys = st.block(0, T)
    W0 = [l.W.astype(np.float64) for l in m.dense_layers]
    pipe = engine.Pipeline(m, counts, "sgd", lr, xs[0] if M > 1 else xs[0, 0], ys[0] if M > 1 else ys[0, 0],
                           act_delay=act_delay, learn=learn, grid=grid)
    outs, losses, valid = pipe.run(xs.astype(np.float32), ys.astype(np.float32))
    got = pipe.extract_weights()
    pipe.close()
    o64, l64, v64, W64, b64 = run_oracle(m, counts, xs, ys, lr, np.float64, act_delay, learn)
    o32, l32, v32, W32, b32 = run_oracle(m, counts, xs, ys, lr, np.float32, act_delay, learn)
    assert np.array_equal(valid.astype(bool), v64)
    vm = v64
    e_out = rel(outs.reshape(o64.shape), o64)
    e_out32 = rel(o32, o64)
    assert e_out <= max(4 * e_out32, 1e-6) or e_out <= 1e-4, (e_out, e_out32)
    if learn:
        e_loss = rel(losses[vm], l64[vm])
        e_loss32 = rel(l32[vm], l64[vm])
        assert e_loss <= max(4 * e_loss32, 1e-6) or e_loss <= 1e-4, (e_loss, e_loss32)
        for j, l in enumerate(got.dense_layers):
            dW = l.W.astype(np.float64) - W0[j]
            dW64 = W64[j] - W0[j]
            if np.linalg.norm(dW64) > 0:
                e = frob_rel(dW, dW64)
                e32 = frob_rel(W32[j] - W0[j], dW64)
                assert e <= max(4 * e32, 1e-6) or e <= 1e-3, (j, e, e32)
            assert frob_rel(l.b, b64[j]) <= 1e-4
    return e_out


@pytest.mark.parametrize("D", [1, 2, 3])
def test_tiny_relu(D):
    counts = {1: [5], 2: [2, 3], 3: [2, 2, 1]}[D]
    _case([5, 7, 6, 3], counts, 30, 0.05)


def test_tiny_tanh_D2():
    _case([6, 9, 8, 4], [2, 3], 30, 0.05, act="tanh")


@pytest.mark.parametrize("act_delay", [0, 1])
def test_act_delay(act_delay):
    _case([16, 24, 24, 8], [2, 3], 40, 0.05, act_delay=act_delay)


def test_c1_8x512_D2():
    """Config 1 (BASELINE.json): 8-layer 512-wide ReLU MLP, batch 1, D=2."""
    _case([512] * 9, [8, 7], 200, 1e-3)


def test_inference_wave():
    _case([64, 128, 128, 64], [2, 3], 20, 0.0, learn=False)


def test_small_grid_uneven_rows():
    _case([40, 130, 70, 9], [2, 3], 25, 0.05, grid=3)


@pytest.mark.parametrize("M", [2, 4])
def test_microbatch_generic(M):
    _case([32, 48, 40, 16], [2, 3], 25, 0.05, M=M)
