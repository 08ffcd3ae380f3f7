import sys; sys.path.insert(0, "/root/repo")
import numpy as np
from paper_2210_09147_b200 import engine, model as mdl, streams
from tests.helpers import run_oracle, rel
widths, counts, T, M = [256, 512, 512, 256, 256], [4, 3], 12, 16
st = streams.SmoothStream(widths[0], widths[-1], seed=5, batch=M)
xs, ys = st.block(0, T)
m = mdl.mlp(widths, seed=4)
o64, *_ = run_oracle(m, counts, xs, ys, 0.05, np.float64)
o32, *_ = run_oracle(m, counts, xs, ys, 0.05, np.float32)
print("oracle f32 vs f64 rel", rel(o32, o64))
for g in (0, 64, 32, 148):
    p = engine.Pipeline(mdl.mlp(widths, seed=4), counts, "sgd", 0.05, xs[0], ys[0], grid=g)
    o, l, v = p.run(xs.astype(np.float32), ys.astype(np.float32))
    print("grid", g, p.kernel_path, "rel vs f64", rel(o.reshape(o64.shape), o64))
    p.close()
