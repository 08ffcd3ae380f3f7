import sys; sys.path.insert(0, '.')
import numpy as np
from paper_2210_09147_b200 import engine, model as mdl, streams
from tests.helpers import run_oracle
M = 2
widths = [32, 16, 8]
for T in (1, 2, 3):
    m = mdl.mlp(widths, act="none", seed=0, loss="mse")
    st = streams.SmoothStream(32, 8, seed=1, batch=M)
    xs, ys = st.block(0, T)
    p = engine.Pipeline(m, [2], "adam", 1e-3, xs[0], ys[0])
    o, l, v = p.run(xs.astype(np.float32), ys.astype(np.float32))
    o64, l64, v64, W64, b64 = run_oracle(m, [2], xs, ys, 1e-3, np.float64, 1, True, "mse", "adam")
    got = p.extract_weights().dense_layers
    for j in range(2):
        W0 = m.dense_layers[j].W.astype(np.float64)
        print("T", T, "layer", j, "W err %.2e" % np.max(np.abs(got[j].W - W64[j])), "b err %.2e" % np.max(np.abs(got[j].b - b64[j])),
              "dW %.2e" % np.max(np.abs(W64[j] - W0)))
    p.close()
for T in (1, 2):
    m = mdl.mlp(widths, act="none", seed=0, loss="mse")
    st = streams.SmoothStream(32, 8, seed=1, batch=M)
    xs, ys = st.block(0, T)
    p = engine.Pipeline(m, [2], "adam", 1e-3, xs[0], ys[0])
    o, l, v = p.run(xs.astype(np.float32), ys.astype(np.float32))
    o64, l64, v64, W64, b64 = run_oracle(m, [2], xs, ys, 1e-3, np.float64, 1, True, "mse", "adam")
    got = p.extract_weights().dense_layers
    b0 = m.dense_layers[1].b.astype(np.float64)
    print("T", T, "gpu db", np.round((got[1].b - b0) * 1e3, 4))
    print("T", T, "ref db", np.round((b64[1] - b0) * 1e3, 4))
    print("   out gpu-ref", np.max(np.abs(o - o64)))
    p.close()
