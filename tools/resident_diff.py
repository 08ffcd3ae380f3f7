"""Where does a resident-step sequence first differ from one pt_run? Runs variants of the
interleaving and prints the first tick whose output differs (bitwise)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2210_09147_b200 import engine, model as mdl, streams

widths, T = [48, 80, 80, 80, 10], 30
D = int(sys.argv[1]) if len(sys.argv) > 1 else 3
counts = {1: [7], 2: [4, 3], 3: [2, 2, 3]}[D]
m = mdl.mlp(widths, seed=7)
xs, ys = streams.SmoothStream(widths[0], widths[-1], seed=8).block(0, T)
xs, ys = xs.astype(np.float32), ys.astype(np.float32)
mk = lambda: engine.Pipeline(m, counts, "sgd", 0.05, xs[0, 0], ys[0, 0])
a = mk()
o_ref, l_ref, _ = a.run(xs, ys)
for name, plan in [("steps", [(30, "step")]), ("steps-run", [(5, "step"), (25, "run")]),
                   ("run-steps", [(5, "run"), (25, "step")]), ("step-get-step", [(5, "step"), (0, "get"), (25, "step")]),
                   ("run-get-run", [(5, "run"), (0, "get"), (25, "run")]), ("runs", [(5, "run"), (25, "run")])]:
    b = mk()
    outs, t = [], 0
    for seg, kind in plan:
        if kind == "get":
            W, bb = b.get_layer(1)
            b.set_layer(1, W, bb)
        elif kind == "run":
            o, l, _ = b.run(xs[t:t + seg], ys[t:t + seg])
            outs += list(o[:, 0])
        else:
            for k in range(seg):
                outs.append(b.step(xs[t + k, 0], ys[t + k, 0]).output)
        t += seg
    outs = np.array(outs)
    bad = [i for i in range(T) if not np.array_equal(outs[i], o_ref[i, 0])]
    print(f"D={D} {name}: first differing tick {bad[0] if bad else None} ({len(bad)} differ), "
          f"max |diff| {np.max(np.abs(outs - o_ref[:, 0])):.3e}", flush=True)
    b.close()
