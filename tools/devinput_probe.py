"""Single process, no time-slicing: a run fed CUDA tensors must equal a run fed numpy arrays
(batch 4 tick kernel and batch 16 tile kernel), repeated."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2210_09147_b200 import engine, model as mdl, streams

for widths, M in (([64, 96, 96, 96, 32], 4), ([256, 512, 512, 256, 256], 16), ([32, 64, 64, 64, 16], 1)):
    T = 40
    st = streams.SmoothStream(widths[0], widths[-1], seed=5, batch=M)
    xs, ys = st.block(0, T)
    xs, ys = xs.astype(np.float32), ys.astype(np.float32)
    s0 = (lambda a: a[0]) if M > 1 else (lambda a: a[0, 0])
    ref = engine.Pipeline(mdl.mlp(widths, seed=4), [4, 3], "sgd", 0.05, s0(xs), s0(ys))
    o_ref, _, _ = ref.run(xs, ys)
    path = ref.kernel_path
    ref.close()
    res = []
    for trial in range(6):
        p = engine.Pipeline(mdl.mlp(widths, seed=4), [4, 3], "sgd", 0.05, s0(xs), s0(ys))
        if trial % 2:
            o, _, _ = p.run(xs, ys)
        else:
            o, _, _ = p.run(torch.from_numpy(xs).cuda(), torch.from_numpy(ys).cuda())
            p.sync()
            o = o.cpu().numpy()
        bad = [t for t in range(T) if not np.array_equal(o[t], o_ref[t])]
        res.append("ok" if not bad else f"BAD@{bad[0]}")
        p.close()
    print(f"M={M} path={path}: {res}", flush=True)
