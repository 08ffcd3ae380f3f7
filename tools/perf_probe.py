"""Quick perf probe: kernel time per tick for a few configs (not the bench)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2210_09147_b200 import engine, model as mdl, streams

def probe(widths, D, learn=True, M=1, ticks=64, reps=3, lr=1e-3):
    m = mdl.mlp(widths, seed=0)
    nl = len(m.layers)
    # equal split over fused units -> module counts
    L = len(widths) - 1
    per = [L // D + (1 if i < L % D else 0) for i in range(D)]
    counts, u = [], 0
    for c in per:
        mods = sum(2 if (u + j) < L - 1 else 1 for j in range(c)); counts.append(mods); u += c
    st = streams.SmoothStream(widths[0], widths[-1], seed=1, batch=M)
    xs, ys = st.block(0, ticks)
    xs = torch.tensor(xs, dtype=torch.float32, device="cuda"); ys = torch.tensor(ys, dtype=torch.float32, device="cuda")
    p = engine.Pipeline(m, counts, "sgd", lr, xs[0].cpu().numpy() if M > 1 else xs[0, 0].cpu().numpy(),
                        ys[0].cpu().numpy() if M > 1 else ys[0, 0].cpu().numpy(), learn=learn)
    per_w = 12 if learn else 4
    bytes_tick = sum(per_w * widths[i] * widths[i + 1] for i in range(L))
    p.run(xs, ys); p.sync()
    best = 1e9
    for _ in range(reps):
        p.run(xs, ys); p.sync(); best = min(best, p.last_kernel_ms())
    us = best * 1e3 / ticks
    print(f"widths={widths[0]}x{L} D={D} M={M} learn={learn}: {us:.1f} us/tick, "
          f"{bytes_tick / (us * 1e-6) / 1e9:.0f} GB/s algorithmic ({bytes_tick/1e6:.0f} MB/tick)", flush=True)
    p.close()

if __name__ == "__main__":
    probe([2048] * 33, 1)
    probe([2048] * 33, 8)
    probe([2048] * 33, 1, learn=False)
    probe([4096] * 17, 1, ticks=32)
    probe([1024] * 33, 1)
    probe([512] * 9, 2, ticks=256)
