"""Cross-CTA skew: every CTA's completion time of every F/B step (pt_set_trace(-1))."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2210_09147_b200 import engine, model as mdl, streams, _lib
import ctypes

def run(widths=[2048] * 33, ticks=4, lr=1e-3):
    m = mdl.mlp(widths, seed=0)
    L = len(widths) - 1
    st = streams.SmoothStream(widths[0], widths[-1], seed=1)
    xs, ys = st.block(0, ticks)
    xs = torch.tensor(xs, dtype=torch.float32, device="cuda"); ys = torch.tensor(ys, dtype=torch.float32, device="cuda")
    p = engine.Pipeline(m, [2 * L - 1], "sgd", lr, xs[0, 0].cpu().numpy(), ys[0, 0].cpu().numpy())
    p.run(xs, ys); p.sync()
    G = 148
    cap = G * 2 * L * ticks
    _lib.check(p._lib.pt_set_trace(p._h, -1, cap))
    p.run(xs, ys); p.sync()
    buf = np.zeros(cap, np.uint64)
    _lib.check(p._lib.pt_get_trace(p._h, buf.ctypes.data_as(ctypes.c_void_p), cap))
    T = buf.reshape(-1, G).astype(np.int64)
    T = T[(T > 0).all(axis=1)]
    rel = (T - T.min(axis=1, keepdims=True)) / 1e3  # us after the first CTA finished the step
    spread = rel.max(axis=1)
    print(f"steps {len(T)}: completion spread median {np.median(spread):.2f} us, p90 {np.percentile(spread, 90):.2f} us")
    rank = np.argsort(np.argsort(T, axis=1), axis=1)
    late = (rank >= G - 8).mean(axis=0)  # how often each CTA is among the last 8
    order = np.argsort(-late)
    print("CTAs most often among the last 8:", [(int(c), round(float(late[c]), 2)) for c in order[:12]])
    print("mean lateness (us) by CTA, top:", [(int(c), round(float(rel[:, c].mean()), 2)) for c in np.argsort(-rel.mean(0))[:12]])
    print("mean lateness (us) by CTA, bottom:", [(int(c), round(float(rel[:, c].mean()), 2)) for c in np.argsort(rel.mean(0))[:6]])
    # F steps vs B steps
    nF = L
    steps = rel.reshape(ticks, 2 * L, G) if len(T) == ticks * 2 * L else None
    if steps is not None:
        print(f"F-step spread median {np.median(steps[:, :L].max(-1)):.2f} us, B-step {np.median(steps[:, L:].max(-1)):.2f} us")
        rows = np.array([int(2048 * (c + 1) / G) - int(2048 * c / G) for c in range(G)])
        for r in (13, 14):
            print(f"  CTAs with {r} rows: mean lateness F {steps[:, :L, rows == r].mean():.2f} B {steps[:, L:, rows == r].mean():.2f}")
    p.close()

if __name__ == "__main__":
    print("lr=1e-3"); run()
    print("lr=0 (no weight write-back)"); run(lr=0.0)
