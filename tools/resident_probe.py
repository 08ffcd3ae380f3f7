"""Resident pt_step (pt_panel.cuh PParams::resident) interleaved with pt_run and weight
reads, printing every call before it is made (a hang shows where). Usage:
resident_probe.py [D] [loss]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2210_09147_b200 import engine, model as mdl, streams

D = int(sys.argv[1]) if len(sys.argv) > 1 else 3
loss = sys.argv[2] if len(sys.argv) > 2 else "mse"
widths = [48, 80, 80, 80, 10]
counts = {1: [7], 2: [4, 3], 3: [2, 2, 3]}[D]
m = mdl.mlp(widths, seed=7, loss=loss)
xs, ys = streams.SmoothStream(widths[0], widths[-1], seed=8).block(0, 30)
if loss == "softmax_ce":
    ys = np.argmax(ys, axis=-1).astype(np.float64)[..., None]
xs, ys = xs.astype(np.float32), ys.astype(np.float32)
p = engine.Pipeline(m, counts, "sgd", 0.05, xs[0, 0], ys[0, 0], timeout_ms=3000)
print("path", p.kernel_path, flush=True)
t = 0
for seg, kind in ((5, "step"), (4, "run"), (7, "step"), (0, "get"), (6, "step"), (8, "run")):
    t1 = time.perf_counter()
    if kind == "get":
        print("get/set layer 1", flush=True)
        W, b = p.get_layer(1)
        p.set_layer(1, W, b)
    elif kind == "run":
        print(f"run [{t}, {t + seg})", flush=True)
        p.run(xs[t:t + seg], ys[t:t + seg])
    else:
        for k in range(seg):
            print(f"step {t + k}", flush=True)
            r = p.step(xs[t + k, 0], ys[t + k, 0])
    print(f"  {kind} done in {1e3 * (time.perf_counter() - t1):.2f} ms", flush=True)
    t += seg
p.close()
print("ok", flush=True)
