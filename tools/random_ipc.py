"""Randomised check of the stage-exchange protocol: two co-resident single-stage handles
(74 CTAs each, CUDA IPC import path) against the single-handle D=2 pipeline on 74 CTAs with
its stages in turn, bit for bit, over random widths, batch and act_delay."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2210_09147_b200 import engine, model as mdl, streams

rng = np.random.default_rng(int(os.environ.get("SEED", "0")))
bad = 0
N = int(os.environ.get("N", "20"))
for k in range(N):
    L = int(rng.integers(2, 6))
    widths = [int(rng.integers(1, int(os.environ.get("WMAX", "600")))) for _ in range(L + 1)]
    cut = int(rng.integers(1, L))
    counts = [2 * cut, 2 * (L - cut) - 1]
    M = int(rng.choice([1, 2, 4]))
    ad = int(rng.integers(0, 2))
    T = int(rng.integers(4, 16))
    st = streams.SmoothStream(widths[0], widths[-1], seed=k, batch=M)
    xs, ys = st.block(0, T)
    xs, ys = xs.astype(np.float32), ys.astype(np.float32)
    s0 = (lambda a: a[0]) if M > 1 else (lambda a: a[0, 0])
    m = mdl.mlp(widths, seed=k)
    a = engine.Pipeline(m, counts, "sgd", 0.05, s0(xs), s0(ys), local_stages=(0, 1), grid=74, act_delay=ad,
                        timeout_ms=60000)
    b = engine.Pipeline(m, counts, "sgd", 0.05, s0(xs), s0(ys), local_stages=(1, 1), grid=74, act_delay=ad,
                        timeout_ms=60000)
    a.ipc_import(b.ipc_export(2))
    b.ipc_import(a.ipc_export(1))
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    a.set_stream(sa)
    b.set_stream(sb)
    xd, yd = torch.from_numpy(xs).cuda(), torch.from_numpy(ys).cuda()
    torch.cuda.synchronize()
    a.run(xd, None, T)
    outs, losses, _ = b.run(None, yd, T)
    a.sync()
    b.sync()
    os.environ["PT_CONC"] = "0"
    ref = engine.Pipeline(m, counts, "sgd", 0.05, s0(xs), s0(ys), grid=74, act_delay=ad)
    os.environ.pop("PT_CONC")
    o, l, _ = ref.run(xs, ys)
    W = [ref.get_layer(j)[0] for j in range(ref.L)]
    mine = [a.get_layer(j)[0] for j in a._local_units()] + [b.get_layer(j)[0] for j in b._local_units()]
    ok = np.array_equal(outs.cpu().numpy(), o) and all(np.array_equal(x, y) for x, y in zip(mine, W))
    if not ok:
        bad += 1
        print(f"case {k} MISMATCH widths {widths} counts {counts} M {M} act_delay {ad} T {T}", flush=True)
    for p in (a, b, ref):
        p.close()
print(f"{bad} / {N} mismatched", flush=True)
