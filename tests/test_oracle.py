"""CPU oracle vs the reference's worked examples and properties (f64).

This pins the oracle: the reference ships no engine, so these are
the only pins. Each test cites the SPEC line it restates.
"""

import numpy as np
import pytest

from oracle import engine as oeng
from oracle import netcore as nc


def rand_net(rng, n_dense, dims=None, acts=("relu", "tanh")):
    dims = dims or [int(rng.integers(2, 9)) for _ in range(n_dense + 1)]
    layers = []
    for i in range(n_dense):
        W = rng.uniform(-1, 1, (dims[i + 1], dims[i]))
        b = rng.uniform(-1, 1, dims[i + 1])
        layers.append(("dense", W, b))
        if i < n_dense - 1:
            layers.append((acts[int(rng.integers(0, len(acts)))],))
    return layers, dims


def clone(layers):
    return [tuple([l[0]] + [np.array(a, copy=True) for a in l[1:]]) for l in layers]


# ---- layer_forward / layer_backward examples ---------------------------------

def test_dense_identity():
    out = nc.layer_forward(("dense", np.eye(2), np.zeros(2)), np.array([[1.0, 2.0]]))
    assert np.array_equal(out, [[1.0, 2.0]])


def test_relu_forward():
    assert np.array_equal(nc.layer_forward(("relu",), np.array([[-1.0, 2.0]])), [[0.0, 2.0]])


def test_dense_derived():
    out = nc.layer_forward(("dense", np.array([[1.0, 1.0], [0.0, 1.0]]), np.zeros(2)), np.array([[1.0, 2.0]]))
    assert np.array_equal(out, [[3.0, 2.0]])


def test_relu_backward():
    g, w = nc.layer_backward(("relu",), np.array([[-1.0, 2.0]]), np.array([[1.0, 1.0]]))
    assert np.array_equal(g, [[0.0, 1.0]]) and w is None


def _fd_check(f, x, grad, h=1e-6):
    num = np.zeros_like(x)
    it = np.nditer(x, flags=["multi_index"])
    for _ in it:
        i = it.multi_index
        xp, xm = x.copy(), x.copy()
        xp[i] += h
        xm[i] -= h
        num[i] = (f(xp) - f(xm)) / (2 * h)
    return np.max(np.abs(num - grad)) / max(np.max(np.abs(num)), 1e-12)


@pytest.mark.parametrize("seed", range(20))
def test_dense_grad_finite_differences(seed):
    """dense weight_grad = outer(upstream, input); input_grad = W^T upstream."""
    rng = np.random.default_rng(seed)
    n_in, n_out, M = (int(v) for v in rng.integers(1, 9, 3))
    W, b = rng.normal(size=(n_out, n_in)), rng.normal(size=n_out)
    x, up = rng.normal(size=(M, n_in)), rng.normal(size=(M, n_out))
    gin, gw = nc.layer_backward(("dense", W, b), x, up)
    assert _fd_check(lambda W_: np.sum(nc.layer_forward(("dense", W_, b), x) * up), W.copy(), gw.dW) <= 1e-5
    assert _fd_check(lambda b_: np.sum(nc.layer_forward(("dense", W, b_), x) * up), b.copy(), gw.db) <= 1e-5
    assert _fd_check(lambda x_: np.sum(nc.layer_forward(("dense", W, b), x_) * up), x.copy(), gin) <= 1e-5
    if M == 1:
        assert np.allclose(gw.dW, np.outer(up[0], x[0]))


@pytest.mark.parametrize("kind", ["relu", "tanh"])
@pytest.mark.parametrize("seed", range(10))
def test_activation_grad_finite_differences(kind, seed):
    rng = np.random.default_rng(seed)
    x = rng.normal(size=(3, 5))
    x[np.abs(x) < 1e-3] = 0.5  # keep away from the relu kink
    up = rng.normal(size=(3, 5))
    gin, _ = nc.layer_backward((kind,), x, up)
    assert _fd_check(lambda x_: np.sum(nc.layer_forward((kind,), x_) * up), x.copy(), gin) <= 1e-5


@pytest.mark.parametrize("seed", range(10))
def test_loss_grad_finite_differences(seed):
    """loss_grad matches central differences of loss_eval; mse(o, o) = 0."""
    rng = np.random.default_rng(seed)
    o, y = rng.normal(size=(2, 4)), rng.normal(size=(2, 4))
    assert _fd_check(lambda o_: nc.loss_eval("mse", o_, y), o.copy(), nc.loss_grad("mse", o, y)) <= 1e-5
    assert nc.loss_eval("mse", o, o) == 0.0
    t = rng.integers(0, 4, 2)
    assert _fd_check(lambda o_: nc.loss_eval("softmax_ce", o_, t), o.copy(), nc.loss_grad("softmax_ce", o, t)) <= 1e-5


def test_softmax_normalises():
    z = np.random.default_rng(0).normal(size=(7, 11)) * 10
    assert np.all(np.abs(nc.softmax(z).sum(-1) - 1) <= 1e-12)


def test_cross_entropy_range_check():
    with pytest.raises(ValueError):
        nc.loss_eval("softmax_ce", np.zeros((1, 3)), np.array([3]))


# ---- sequential_step --------------------------------------------------------

def test_sequential_lr0_bit_identical():
    rng = np.random.default_rng(1)
    layers, dims = rand_net(rng, 3)
    before = clone(layers)
    nc.sequential_step(layers, rng.normal(size=(1, dims[0])), rng.normal(size=(1, dims[-1])), lr=0.0)
    for a, b in zip(layers, before):
        for u, v in zip(a[1:], b[1:]):
            assert np.array_equal(u, v)


def test_sequential_deterministic():
    rng = np.random.default_rng(2)
    layers, dims = rand_net(rng, 4)
    x, y = rng.normal(size=(1, dims[0])), rng.normal(size=(1, dims[-1]))
    a, b = clone(layers), clone(layers)
    o1 = nc.sequential_step(a, x, y, lr=0.1)[0]
    o2 = nc.sequential_step(b, x, y, lr=0.1)[0]
    assert np.array_equal(o1, o2)
    for la, lb in zip(a, b):
        for u, v in zip(la[1:], lb[1:]):
            assert np.array_equal(u, v)


def test_sequential_three_layer_fd():
    """GradientBundle matches finite differences on a 3-layer dense net."""
    rng = np.random.default_rng(3)
    layers, dims = rand_net(rng, 3, acts=("tanh",))
    x, y = rng.normal(size=(1, dims[0])), rng.normal(size=(1, dims[-1]))
    out, inputs = nc.block_forward(layers, x)
    _, grads = nc.block_backward(layers, inputs, nc.loss_grad("mse", out, y))
    for j, l in enumerate(layers):
        if l[0] != "dense":
            continue

        def f(W_, j=j):
            ls = clone(layers)
            ls[j] = ("dense", W_, ls[j][2])
            return nc.loss_eval("mse", nc.forward_only(ls, x), y)
        assert _fd_check(f, l[1].copy(), grads[j].dW) <= 1e-5


def test_sequential_nonfinite_raises_with_step():
    layers = [("dense", np.array([[np.inf]]), np.zeros(1))]
    with pytest.raises(FloatingPointError, match="step 7"):
        nc.sequential_step(layers, np.ones((1, 1)), np.zeros((1, 1)), lr=0.1, step_index=7)


# ---- engine ---------------------------------------------------------------

def _bounds_for(layers, D, rng):
    """Random contiguous plan over dense units (activations stay with their dense layer)."""
    starts = [i for i, l in enumerate(layers) if l[0] == "dense"]
    cut = sorted(rng.choice(np.arange(1, len(starts)), D - 1, replace=False)) if D > 1 else []
    return [0] + [starts[c] for c in cut] + [len(layers)]


@pytest.mark.parametrize("D", [1, 2, 3, 4])
@pytest.mark.parametrize("seed", range(5))
def test_output_delay_invariant(D, seed):
    """lr=0: output(t) = f(x^(t-(D-1))) for t >= D-1 (Eq. 7, acceptance #1)."""
    rng = np.random.default_rng(100 + seed)
    layers, dims = rand_net(rng, int(rng.integers(D, 7)))
    bounds = _bounds_for(layers, D, rng)
    xs = rng.normal(size=(20, 1, dims[0]))
    ys = rng.normal(size=(20, 1, dims[-1]))
    p = oeng.Pipeline(clone(layers), bounds, 0.0, xs[0], ys[0])
    for t in range(20):
        o = p.step(xs[t], ys[t])
        assert o.valid == (t >= D - 1) and o.source_sample_id == t - (D - 1)
        if o.valid:
            ref = nc.forward_only(layers, xs[t - D + 1])
            assert np.max(np.abs(o.output - ref)) <= 1e-12
            assert abs(o.loss - nc.loss_eval("mse", ref, ys[t - D + 1])) <= 1e-12


@pytest.mark.parametrize("act_delay", [0, 1])
@pytest.mark.parametrize("D", [2, 3, 4])
def test_constant_stream_gradients(D, act_delay):
    """lr=0, constant stream: stage h's gradients equal the oracle's slice for t >= 2D-h-1
    (Eq. 9-10, acceptance #2), for both delay readings."""
    rng = np.random.default_rng(7 * D + act_delay)
    layers, dims = rand_net(rng, 6)
    bounds = _bounds_for(layers, D, rng)
    x, y = rng.normal(size=(1, dims[0])), rng.normal(size=(1, dims[-1]))
    out, inputs = nc.block_forward(layers, x)
    _, ref = nc.block_backward(layers, inputs, nc.loss_grad("mse", out, y))
    p = oeng.Pipeline(clone(layers), bounds, 0.0, x, y, act_delay=act_delay)
    for t in range(3 * D + 2):
        p.step(x, y)
        for h in range(1, D + 1):
            if t >= 2 * D - h - 1:
                for j, g in enumerate(p.last_grads[h]):
                    if g is not None:
                        r = ref[bounds[h - 1] + j]
                        assert np.max(np.abs(g.dW - r.dW)) <= 1e-12
                        assert np.max(np.abs(g.db - r.db)) <= 1e-12


def test_literal_prev_cache_reading_would_fail_criterion_2():
    """backpropagating stage D through the previous tick's cache breaks
    acceptance #2 at (h=D, t=D-1); the SPEC reading keeps stage D on the current tick."""
    rng = np.random.default_rng(5)
    layers, dims = rand_net(rng, 4)
    D = 2
    bounds = _bounds_for(layers, D, rng)
    x, y = rng.normal(size=(1, dims[0])), rng.normal(size=(1, dims[-1]))
    out, inputs = nc.block_forward(layers, x)
    _, ref = nc.block_backward(layers, inputs, nc.loss_grad("mse", out, y))
    # literal reading: stage D uses cache[(t-1)%2] -> at t = D-1 that cache is still zero
    p = oeng.Pipeline(clone(layers), bounds, 0.0, x, y)
    p.step(x, y)
    st = p.stages[-1]
    stale_inputs = st.cache[(D - 1 - 1) % 2]
    o = nc.forward_only(st.layers, p.stages[-1].inslot[(D - 1) % 2] if D > 1 else x)
    _, lit = nc.block_backward(st.layers, stale_inputs, nc.loss_grad("mse", o, y))
    dense_lit = [g for g in lit if g is not None]
    dense_ref = [g for g in ref[bounds[-2]:] if g is not None]
    assert any(np.max(np.abs(a.dW - b.dW)) > 1e-6 for a, b in zip(dense_lit, dense_ref))


@pytest.mark.parametrize("seed", range(5))
def test_d1_equivalence_with_updates(seed):
    """D=1 pipeline == sequential_step step for step, including updates."""
    rng = np.random.default_rng(200 + seed)
    layers, dims = rand_net(rng, 5)
    xs, ys = rng.normal(size=(15, 1, dims[0])), rng.normal(size=(15, 1, dims[-1]))
    p = oeng.Pipeline(clone(layers), [0, len(layers)], 0.05, xs[0], ys[0])
    seq = clone(layers)
    for t in range(15):
        o = p.step(xs[t], ys[t])
        so, sl, _ = nc.sequential_step(seq, xs[t], ys[t], lr=0.05)
        assert np.max(np.abs(o.output - so)) <= 1e-12 and abs(o.loss - sl) <= 1e-12
    for a, b in zip(p.extract_weights(), seq):
        for u, v in zip(a[1:], b[1:]):
            assert np.max(np.abs(u - v)) <= 1e-12


def test_buffer_safety():
    """The payload stage h writes at step t is the one stage h+1 reads at t+1."""
    rng = np.random.default_rng(9)
    layers, dims = rand_net(rng, 4)
    D = 3
    bounds = _bounds_for(layers, D, rng)
    p = oeng.Pipeline(clone(layers), bounds, 0.01, np.zeros((1, dims[0])), np.zeros((1, dims[-1])))
    seen = {}
    orig = oeng.Pipeline._stage_tick

    def spy(self, st, t, x_t, res):
        if st.h > 1:
            seen[(st.h, t)] = st.inslot[(t - 1) % 2].copy()
        orig(self, st, t, x_t, res)
        if st.h < self.D:
            seen[("out", st.h, t)] = res[("act", st.h)].copy()
    p._stage_tick = spy.__get__(p, oeng.Pipeline)
    for t in range(8):
        p.step(rng.normal(size=(1, dims[0])), rng.normal(size=(1, dims[-1])))
    for t in range(1, 8):
        for h in range(2, D + 1):
            assert np.array_equal(seen[(h, t)], seen[("out", h - 1, t - 1)])


def test_buffer_swap_mutation_is_caught():
    """Mutation smoke test: an off-by-one in the buffer swap (reading the slot
    written in the same step) breaks the output-delay invariant."""
    rng = np.random.default_rng(11)
    layers, dims = rand_net(rng, 4)
    D = 2
    bounds = _bounds_for(layers, D, rng)
    xs = rng.normal(size=(8, 1, dims[0]))

    class Mutant(oeng.Pipeline):
        def _stage_tick(self, st, t, x_t, res):
            if st.h > 1 and ("act", st.h - 1) in res:  # read this step's payload
                st.inslot[(t - 1) % 2] = res[("act", st.h - 1)]
            super()._stage_tick(st, t, x_t, res)

    m = Mutant(clone(layers), bounds, 0.0, xs[0], np.zeros((1, dims[-1])))
    bad = False
    for t in range(8):
        o = m.step(xs[t], np.zeros((1, dims[-1])))
        if o.valid and np.max(np.abs(o.output - nc.forward_only(layers, xs[t - D + 1]))) > 1e-12:
            bad = True
    assert bad


def test_target_alignment_and_warmup():
    """Stage D pairs output(t) with gamma_{t-(D-1)}; n_steps = D-1 gives no valid output
    (SPEC.md:232, 251)."""
    rng = np.random.default_rng(13)
    layers, dims = rand_net(rng, 4)
    D = 3
    p = oeng.Pipeline(clone(layers), _bounds_for(layers, D, rng), 0.0, np.zeros((1, dims[0])),
                      np.zeros((1, dims[-1])))
    outs = oeng.pipeline_run(p, rng.normal(size=(D - 1, 1, dims[0])), rng.normal(size=(D - 1, 1, dims[-1])), D - 1)
    assert not any(o.valid for o in outs)


@pytest.mark.parametrize("D", [2, 3, 4])
def test_engine_schedule_matches_simulator(D):
    """Engine events == PARTIME simulator events, 50 steps (acceptance #6)."""
    rng = np.random.default_rng(D)
    layers, dims = rand_net(rng, 6)
    p = oeng.Pipeline(clone(layers), _bounds_for(layers, D, rng), 0.01, np.zeros((1, dims[0])),
                      np.zeros((1, dims[-1])), record_events=True)
    for t in range(50):
        p.step(rng.normal(size=(1, dims[0])), rng.normal(size=(1, dims[-1])))
    key = lambda e: (e.slot, e.stage, e.op, e.sample_id)
    assert sorted(map(key, p.events)) == sorted(map(key, oeng.partime_schedule(D, 50)))


def test_schedule_examples():
    """D=3, t=6, h=1 -> F(6), B(2); stage-1 backward 2(D-h)=4 steps after its forward
    (SPEC.md:225, 299)."""
    ev = oeng.partime_schedule(3, 12)
    at = {(e.slot, e.stage, e.op): e.sample_id for e in ev}
    assert at[(6, 1, "F")] == 6 and at[(6, 1, "B")] == 2
    for k in range(5):
        f = next(e.slot for e in ev if e.stage == 1 and e.op == "F" and e.sample_id == k)
        b = next(e.slot for e in ev if e.stage == 1 and e.op == "B" and e.sample_id == k)
        assert b - f == 4


def test_threaded_workers_match_sequential_stage_loop():
    """D workers + 2 barriers per step give identical results."""
    rng = np.random.default_rng(21)
    layers, dims = rand_net(rng, 6)
    D = 3
    bounds = _bounds_for(layers, D, rng)
    xs, ys = rng.normal(size=(12, 1, dims[0])), rng.normal(size=(12, 1, dims[-1]))
    a = oeng.Pipeline(clone(layers), bounds, 0.05, xs[0], ys[0])
    b = oeng.Pipeline(clone(layers), bounds, 0.05, xs[0], ys[0], threads=True)
    for t in range(12):
        oa, ob = a.step(xs[t], ys[t]), b.step(xs[t], ys[t])
        assert np.array_equal(oa.output, ob.output)
    b.close()


def test_concurrent_step_is_a_contract_violation():
    rng = np.random.default_rng(22)
    layers, dims = rand_net(rng, 2)
    p = oeng.Pipeline(clone(layers), [0, len(layers)], 0.0, np.zeros((1, dims[0])), np.zeros((1, dims[-1])))
    p._busy.acquire()
    with pytest.raises(RuntimeError, match="contract violation"):
        p.step(np.zeros((1, dims[0])), np.zeros((1, dims[-1])))


def test_plan_errors():
    layers = [("dense", np.eye(2), np.zeros(2))]
    with pytest.raises(ValueError):
        oeng.Pipeline(layers, [0, 1, 1], 0.0, np.zeros((1, 2)), np.zeros((1, 2)))
    bad = [("dense", np.eye(2), np.zeros(2)), ("dense", np.ones((2, 3)), np.zeros(2))]
    with pytest.raises(ValueError, match="stage boundary 1->2"):
        oeng.Pipeline(bad, [0, 1, 2], 0.0, np.zeros((1, 2)), np.zeros((1, 2)))
