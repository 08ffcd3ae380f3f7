"""Where the per-sample pt_step time goes (C2): wall time per call vs the device time of its
one-tick launch."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2210_09147_b200 import engine, model as mdl, streams

m = mdl.mlp([2048] * 33, seed=0)
st = streams.SmoothStream(2048, 2048, seed=1)
xs, ys = st.block(0, 64)
xs, ys = xs.astype(np.float32), ys.astype(np.float32)
p = engine.Pipeline(m, [len(m.layers)], "sgd", 1e-3, xs[0, 0], ys[0, 0])
for t in range(8):
    p.step(xs[t, 0], ys[t, 0])
wall, dev = [], []
for t in range(32):
    t0 = time.perf_counter()
    p.step(xs[t % 64, 0], ys[t % 64, 0])
    wall.append(time.perf_counter() - t0)
    dev.append(p.last_kernel_ms() * 1e3)
print(f"pt_step wall {np.median(wall) * 1e6:.1f} us, one-tick launch device {np.median(dev):.1f} us")
o = p.run(xs[:16], ys[:16])
p.sync()
print(f"pt_run 16 ticks: device {p.last_kernel_ms() * 1e3 / 16:.1f} us/tick")
p.close()
