"""Single-GPU device time per tick for every BASELINE.json config shape (all stages on one GPU)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2210_09147_b200 import engine, model as mdl, streams, partition

def counts_for(widths, D, learn):
    L = len(widths) - 1
    costs, _ = partition.mlp_costs(widths, learn)
    units, _ = partition.balance(costs, D)
    out, u = [], 0
    for c in units:
        out.append(sum(2 if (u + j) < L - 1 else 1 for j in range(c))); u += c
    return out

def probe(name, widths, D, learn=True, M=1, ticks=16, reps=3):
    m = mdl.mlp(widths, seed=0)
    st = streams.SmoothStream(widths[0], widths[-1], seed=1, batch=M)
    xs, ys = st.block(0, ticks)
    xs = torch.tensor(xs, dtype=torch.float32, device="cuda"); ys = torch.tensor(ys, dtype=torch.float32, device="cuda")
    p = engine.Pipeline(m, counts_for(widths, D, learn), "sgd", 1e-3 if learn else 0.0,
                        xs[0].cpu().numpy() if M > 1 else xs[0, 0].cpu().numpy(),
                        ys[0].cpu().numpy() if M > 1 else ys[0, 0].cpu().numpy(), learn=learn)
    p.run(xs, ys); p.sync()
    best = 1e9
    for _ in range(reps):
        p.run(xs, ys); p.sync(); best = min(best, p.last_kernel_ms())
    us = best * 1e3 / ticks
    per = 12 if learn else 4
    byt = sum(per * widths[i] * widths[i + 1] for i in range(len(widths) - 1))
    print(f"{name}: D={D} M={M} learn={learn}: {us:.1f} us/tick, {M * 1e6 / us:.0f} samples/s, "
          f"{byt / (us * 1e-6) / 1e9:.0f} GB/s algorithmic ({byt / 6500.3e9 * 1e6:.0f} us roofline)", flush=True)
    p.close()

if __name__ == "__main__":
    probe("C1 8x512", [512] * 9, 2, ticks=256)
    probe("C2 32x2048", [2048] * 33, 1, ticks=32)
    probe("C2 32x2048 (D=2 on 1 GPU)", [2048] * 33, 2, ticks=32)
    probe("C3 64x4096 infer", [4096] * 65, 1, learn=False, ticks=8)
    probe("C4 32x4096 M=16", [4096] * 33, 1, M=16, ticks=4, reps=1)
    c5 = [1024, 2048, 4096, 8192, 8192, 4096, 2048, 1024] * 3 + [1024]
    probe("C5 uneven", c5, 2, ticks=8)
