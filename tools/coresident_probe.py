"""Two co-resident stage handles on one GPU (tests/test_gpu_ipc.py setup) with host-side
timings of each call and, on a timeout, the last traced step of every CTA of both handles.
Usage: coresident_probe.py {panel|panel_wide|tile|tick} [reps]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2210_09147_b200 import engine, model as mdl, streams

CASES = {"panel": ([32, 64, 64, 64, 16], [4, 3], 12, 1, 74), "panel_wide": ([256, 512, 512, 512, 128], [4, 3], 40, 1, 74),
         "tile": ([256, 512, 512, 256, 256], [4, 3], 12, 16, 64), "tick": ([32, 64, 64, 64, 16], [4, 3], 12, 1, 74)}
kind = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
if kind == "tick":
    os.environ["PT_PANEL"] = "0"
widths, counts, T, M, grid = CASES[kind]
st = streams.SmoothStream(widths[0], widths[-1], seed=5, batch=M)
xs, ys = st.block(0, T)
xs, ys = xs.astype(np.float32), ys.astype(np.float32)
s0 = (lambda a: a[0]) if M > 1 else (lambda a: a[0, 0])
for rep in range(reps):
    m = mdl.mlp(widths, seed=4)
    a = engine.Pipeline(m, counts, "sgd", 0.05, s0(xs), s0(ys), local_stages=(0, 1), grid=grid, timeout_ms=5000)
    b = engine.Pipeline(m, counts, "sgd", 0.05, s0(xs), s0(ys), local_stages=(1, 1), grid=grid, timeout_ms=5000)
    a.ipc_import(b.ipc_export(2))
    b.ipc_import(a.ipc_export(1))
    for p in (a, b):
        p.set_trace(-1, 4096)
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    a.set_stream(sa)
    b.set_stream(sb)
    xd, yd = torch.from_numpy(xs).cuda(), torch.from_numpy(ys).cuda()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    a.run(xd, None, T)
    t1 = time.perf_counter()
    b.run(None, yd, T)
    t2 = time.perf_counter()
    err = []
    for name, p in (("a", a), ("b", b)):
        try:
            p.sync()
        except Exception as e:  # noqa: BLE001
            err.append(f"{name}: {e}")
    t3 = time.perf_counter()
    print(f"rep {rep} {kind}: a.run {1e3*(t1-t0):.1f} ms, b.run {1e3*(t2-t1):.1f} ms, sync {1e3*(t3-t2):.1f} ms, "
          f"errors {err}", flush=True)
    if err:
        import ctypes
        from paper_2210_09147_b200 import _lib
        for name, p in (("a", a), ("b", b)):
            buf = np.zeros(4096, np.uint64)
            p._lib.pt_get_trace(p._h, buf.ctypes.data_as(ctypes.c_void_p), 4096)
            G = grid if kind != "tile" else 16
            steps = [int(np.count_nonzero(buf[c::G][: 4096 // G])) for c in range(G)]
            print(name, "step ends reached per CTA:", steps, flush=True)
    for p in (a, b):
        p.close()
