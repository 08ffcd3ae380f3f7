import sys; sys.path.insert(0, '.')
import numpy as np
from paper_2210_09147_b200 import engine, model as mdl, streams
from tests.helpers import run_oracle, rel
OPT, LR = sys.argv[1], float(sys.argv[2])
for act in ("none", "relu"):
    for M in (1, 2, 4):
        widths = [32, 48, 40, 8]
        T = 20
        m = mdl.mlp(widths, act=act, seed=0, loss="mse")
        st = streams.SmoothStream(32, 8, seed=1, batch=M)
        xs, ys = st.block(0, T)
        p = engine.Pipeline(m, [5] if act != "none" else [3], OPT, LR, xs[0] if M > 1 else xs[0, 0], ys[0] if M > 1 else ys[0, 0])
        o, l, v = p.run(xs.astype(np.float32), ys.astype(np.float32))
        cnt = [5] if act != "none" else [3]
        o64, *_ = run_oracle(m, cnt, xs, ys, LR, np.float64, 1, True, "mse", OPT)
        o32, *_ = run_oracle(m, cnt, xs, ys, LR, np.float32, 1, True, "mse", OPT)
        print(act, "M", M, "gpu err %.2e" % rel(o, o64), "f32 oracle err %.2e" % rel(o32, o64))
        p.close()
