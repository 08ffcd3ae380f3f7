"""One small run of a kernel path, for compute-sanitizer (racecheck / synccheck / memcheck).
Usage: compute-sanitizer --tool racecheck python tools/sanitize_one.py {panel|tick|tile}"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2210_09147_b200 import engine, model as mdl, streams

kind = sys.argv[1]
if kind == "tick":
    os.environ["PT_PANEL"] = "0"
widths, counts, M = {"panel": ([64, 96, 96, 32], [2, 3], 1), "tick": ([64, 96, 96, 32], [2, 3], 1),
                     "tile": ([256, 256, 256], [2, 1], 16)}[kind]
st = streams.SmoothStream(widths[0], widths[-1], seed=1, batch=M)
xs, ys = st.block(0, 4)
xs, ys = xs.astype(np.float32), ys.astype(np.float32)
p = engine.Pipeline(mdl.mlp(widths, seed=0), counts, "sgd", 0.01, xs[0] if M > 1 else xs[0, 0],
                    ys[0] if M > 1 else ys[0, 0], grid=8 if kind != "tile" else 0, timeout_ms=600000)
assert p.kernel_path == kind, p.kernel_path
o, l, v = p.run(xs, ys)
print(kind, "ok", float(np.abs(o).sum()))
p.close()
