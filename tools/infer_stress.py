"""Repeat test_inference_wave's case (D=2, inference, tick kernel) and localise any run that
differs from the f64 oracle: which ticks, which output rows, and what the wrong values look like."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2210_09147_b200 import engine, model as mdl, streams
from tests.helpers import rel, run_oracle

widths, counts, T = [64, 128, 128, 64], [2, 3], 20
learn = os.environ.get("LEARN", "0") == "1"
m = mdl.mlp(widths, seed=0)
st = streams.SmoothStream(widths[0], widths[-1], seed=1)
xs, ys = st.block(0, T)
o64, *_ = run_oracle(m, counts, xs, ys, 0.0, np.float64, learn=learn)
o64 = o64.reshape(T, -1)
bad_runs = 0
for k in range(int(os.environ.get("N", "60"))):
    p = engine.Pipeline(m, counts, "sgd", 0.0, xs[0, 0], ys[0, 0], learn=learn)
    o, l, v = p.run(xs.astype(np.float32), ys.astype(np.float32))
    p.close()
    o = o.reshape(T, -1)
    err = np.abs(o - o64).max(axis=1) / (np.abs(o64).max() + 1e-30)
    bad = np.nonzero(err > 1e-4)[0]
    if bad.size:
        bad_runs += 1
        t0 = bad[0]
        # is the wrong output the oracle output of another tick (stale or early input)?
        match = [s for s in range(T) if np.abs(o[t0] - o64[s]).max() / (np.abs(o64).max()) < 1e-4]
        print(f"run {k}: bad ticks {bad.tolist()} err {err[t0]:.3g}; tick {t0} output equals oracle tick(s) {match}; "
              f"zeros {np.count_nonzero(o[t0] == 0)}/{o.shape[1]}", flush=True)
print(f"{bad_runs} bad runs", flush=True)
