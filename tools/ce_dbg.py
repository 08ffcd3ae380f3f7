import sys; sys.path.insert(0, '.')
import numpy as np
from paper_2210_09147_b200 import engine, model as mdl, streams
from tests.helpers import run_oracle
for M, D, counts in ((4, 1, [5]), (1, 1, [5]), (2, 1, [5])):
    widths = [32, 48, 40, 8]
    m = mdl.mlp(widths, seed=0, loss="mse")
    st = streams.SmoothStream(32, 8, seed=1, batch=M)
    xs, ys = st.block(0, 20)
    p = engine.Pipeline(m, counts, "adam", 1e-3, xs[0] if M > 1 else xs[0, 0], ys[0] if M > 1 else ys[0, 0])
    o, l, v = p.run(xs.astype(np.float32), ys.astype(np.float32))
    o64, l64, v64, W64, b64 = run_oracle(m, counts, xs, ys, 1e-3, np.float64, 1, True, "mse", "adam")
    print("M", M, "D", D, "out err per tick", ["%.1e" % float(np.max(np.abs(o[t] - o64[t]))) for t in range(20)])
    print("  W err", ["%.1e" % float(np.max(np.abs(a.W - b))) for a, b in zip(p.extract_weights().dense_layers, W64)])
