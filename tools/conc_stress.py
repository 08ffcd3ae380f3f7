"""Repeat the C2-shape D=2 parity case (concurrent stages on 74 + 74 CTAs) against the f64 oracle."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2210_09147_b200 import engine, model as mdl, streams
from tests.helpers import rel, run_oracle

widths, counts, T, lr = [2048] * 33, [32, 31], 5, 1e-3
m = mdl.mlp(widths, seed=0)
st = streams.SmoothStream(widths[0], widths[-1], seed=1)
xs, ys = st.block(0, T)
o64, *_ = run_oracle(m, counts, xs, ys, lr, np.float64)
ref = None
for k in range(int(os.environ.get("N", "12"))):
    p = engine.Pipeline(m, counts, "sgd", lr, xs[0, 0], ys[0, 0])
    o, l, v = p.run(xs.astype(np.float32), ys.astype(np.float32))
    p.close()
    e = rel(o.reshape(o64.shape), o64)
    same = ref is None or np.array_equal(o, ref)
    if ref is None:
        ref = o
    print(f"run {k}: rel err {e:.2e} bitwise-same-as-first {same}", flush=True)
