"""Engine/simulator schedule agreement (acceptance 6 at SPEC.md:466), with the
engine's schedule OBSERVED on the device rather than restated.

Every stage is one linear unit with W = I and the targets are 0, so sample k's output error
is proportional to x_k, a one-hot at position k. The weight change stage h applies at tick t
is then -lr delta a^T with delta ~ e_kb: its row reveals which sample's gradient the
device paired with tick t (B_h(t)), its column which sample's stage input it used
(the act_delay pairing), and the output at tick t reveals F_D(t). These observed events must
equal engine.timeline() and schedsim.simulate(partime) event for event.
"""

import numpy as np
import pytest

from paper_2210_09147_b200 import engine, model as mdl, schedsim

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("D", [2, 3, 4])
@pytest.mark.parametrize("act_delay", [0, 1])
def test_device_schedule_matches_simulator(D, act_delay):
    n = 8
    T = n + 2 * D - 2
    d = 32
    m = mdl.mlp([d] * (D + 1), act="none", seed=0)
    for l in m.dense_layers:
        l.W[:] = np.eye(d, dtype=np.float32)
        l.b[:] = 0
    lr = 1e-3
    xs = np.zeros((T, d), np.float32)
    xs[np.arange(T), np.arange(T)] = 1.0
    ys = np.zeros((T, d), np.float32)
    p = engine.Pipeline(m, [1] * D, "sgd", lr, xs[0], ys[0], act_delay=act_delay)
    prev = [p.get_layer(j)[0].astype(np.float64) for j in range(D)]
    observed = []
    for t in range(T):
        o = p.step(xs[t], ys[t])
        if t - (D - 1) >= 0:
            assert o.valid and int(np.argmax(o.output)) == t - (D - 1)  # F_D(t), on the device
            if t - (D - 1) < n:
                observed.append(("F", t, D, t - (D - 1)))
        for j in range(D):
            W = p.get_layer(j)[0].astype(np.float64)
            dW = W - prev[j]
            prev[j] = W
            h = j + 1
            if np.max(np.abs(dW)) == 0:
                continue  # warm-up: no update on the device
            r, c = np.unravel_index(np.argmax(np.abs(dW)), dW.shape)
            # the gradient's sample, and the stage-input sample it was paired with
            if r < n:
                observed.append(("B", t, h, int(r)))
            want_c = (t - (h - 1)) if (act_delay == 0 or h == D) else (t - 1 - (h - 1))
            assert c == want_c, (t, h, r, c, want_c)
    p.close()
    sim, _ = schedsim.simulate(schedsim.SchedulePolicy("partime", D, n))
    sim_b = sorted((e.op, e.slot, e.stage, e.sample) for e in sim if e.op == "B")
    sim_fD = sorted((e.op, e.slot, e.stage, e.sample) for e in sim if e.op == "F" and e.stage == D)
    got_b = sorted(e for e in observed if e[0] == "B")
    got_fD = sorted(e for e in observed if e[0] == "F")
    assert got_b == sim_b
    assert got_fD == sim_fD
    # and the engine's own record agrees with the simulator on every event
    p2 = engine.Pipeline(m, [1] * D, "sgd", lr, xs[0], ys[0], act_delay=act_delay)
    p2.run(xs, ys)
    p2.sync()
    eng = sorted((e.slot, e.stage, e.op, e.sample) for e in p2.timeline(n))
    p2.close()
    assert eng == sorted((e.slot, e.stage, e.op, e.sample) for e in sim)
