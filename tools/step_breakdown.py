"""Per-call cost of the per-sample path on a tiny model (C1-like), split into Python layer,
C-ABI call and device time."""
import os, sys, time, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2210_09147_b200 import engine, model as mdl, streams, _lib

for widths in ([512] * 9, [2048] * 33):
    m = mdl.mlp(widths, seed=0)
    st = streams.SmoothStream(widths[0], widths[-1], seed=1)
    xs, ys = st.block(0, 64)
    xs, ys = xs.astype(np.float32), ys.astype(np.float32)
    p = engine.Pipeline(m, [len(m.layers)], "sgd", 1e-3, xs[0, 0], ys[0, 0])
    for t in range(8):
        p.step(xs[t, 0], ys[t, 0])
    N = 64
    t0 = time.perf_counter()
    for t in range(N):
        p.step(xs[t, 0], ys[t, 0])
    py = (time.perf_counter() - t0) / N
    dev = p.last_kernel_ms() * 1e3
    out = np.empty(widths[-1], np.float32); loss = np.empty(1, np.float32); valid = np.empty(1, np.uint8)
    x = np.ascontiguousarray(xs[0, 0]); y = np.ascontiguousarray(ys[0, 0])
    t0 = time.perf_counter()
    for t in range(N):
        p._lib.pt_step(p._h, x.ctypes.data_as(ctypes.c_void_p), y.ctypes.data_as(ctypes.c_void_p),
                       out.ctypes.data_as(ctypes.c_void_p), loss.ctypes.data_as(ctypes.c_void_p),
                       valid.ctypes.data_as(ctypes.c_void_p), _lib.PT_HOST)
    c = (time.perf_counter() - t0) / N
    o = p.run(xs, ys)
    p.sync()
    run_us = p.last_kernel_ms() * 1e3 / 64
    print(f"{len(widths)-1}x{widths[0]}: Pipeline.step {py*1e6:.1f} us, raw pt_step {c*1e6:.1f} us, "
          f"one-tick launch device {dev:.1f} us, pt_run device {run_us:.1f} us/tick", flush=True)
    p.close()
