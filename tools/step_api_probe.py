"""Per-sample API cost (engine.Pipeline.step -> pt_step, host buffers): resident launch vs one
launch per step (PT_RESIDENT=0, set per process), against the device tick time of pt_run.
Usage: step_api_probe.py [width] [layers] [calls]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2210_09147_b200 import engine, model as mdl, streams

W = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
L = int(sys.argv[2]) if len(sys.argv) > 2 else 32
N = int(sys.argv[3]) if len(sys.argv) > 3 else 200
m = mdl.mlp([W] * (L + 1), seed=0)
xs, ys = streams.SmoothStream(W, W, seed=1).block(0, 64)
xs, ys = xs.astype(np.float32), ys.astype(np.float32)
p = engine.Pipeline(m, [len(m.layers)], "sgd", 1e-3, xs[0, 0], ys[0, 0])
p.run(xs, ys)
p.run(xs, ys)
p.sync()
tick_us = p.last_kernel_ms() * 1e3 / 64
for _ in range(10):
    p.step(xs[0, 0], ys[0, 0])
t0 = time.perf_counter()
for i in range(N):
    p.step(xs[i % 64, 0], ys[i % 64, 0])
el = (time.perf_counter() - t0) / N * 1e6
x0, y0 = xs[0, 0], ys[0, 0]
t0 = time.perf_counter()
for i in range(N):
    p._lib.pt_step(p._h, x0.ctypes.data, y0.ctypes.data, None, None, None, 0)
raw = (time.perf_counter() - t0) / N * 1e6
print(f"{L}x{W} PT_RESIDENT={os.environ.get('PT_RESIDENT', '1')}: tick {tick_us:.1f} us (pt_run), "
      f"Pipeline.step {el:.1f} us/call, raw pt_step {raw:.1f} us/call", flush=True)
p.close()
