"""Tick time vs grid size (CTAs) for C1 and C2 (tick kernel)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2210_09147_b200 import engine, model as mdl, streams


def probe(name, widths, counts, grid, ticks):
    m = mdl.mlp(widths, seed=0)
    st = streams.SmoothStream(widths[0], widths[-1], seed=1)
    xs, ys = st.block(0, ticks)
    xs = torch.tensor(xs, dtype=torch.float32, device="cuda"); ys = torch.tensor(ys, dtype=torch.float32, device="cuda")
    p = engine.Pipeline(m, counts, "sgd", 1e-3, xs[0, 0].cpu().numpy(), ys[0, 0].cpu().numpy(), grid=grid)
    p.run(xs, ys); p.sync()
    best = 1e9
    for _ in range(3):
        p.run(xs, ys); p.sync(); best = min(best, p.last_kernel_ms())
    print(f"{name} grid {grid}: {best * 1e3 / ticks:.1f} us/tick", flush=True)
    p.close()


if __name__ == "__main__":
    for g in (148, 96, 64, 32, 16, 8):
        probe("C1 8x512 D=2", [512] * 9, [8, 7], g, 256)
    for g in (148, 140, 128, 112, 96, 74):
        probe("C2 32x2048 D=1", [2048] * 33, [63], g, 32)
