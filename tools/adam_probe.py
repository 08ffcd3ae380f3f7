"""Device time per tick of C2 (32 x 2048, batch 1) with Adam (tick kernel) and SGD (panel
kernel), against their roofline (28 / 12 B per weight per tick)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2210_09147_b200 import engine, model as mdl, streams

W, L, T = 2048, 32, 32
m = mdl.mlp([W] * (L + 1), seed=0)
xs, ys = streams.SmoothStream(W, W, seed=1).block(0, T)
xs = torch.tensor(xs, dtype=torch.float32, device="cuda")
ys = torch.tensor(ys, dtype=torch.float32, device="cuda")
for opt in ("sgd", "adam"):
    p = engine.Pipeline(m, [2 * L - 1], opt, 1e-3 if opt == "sgd" else 1e-4, xs[0, 0].cpu().numpy(), ys[0, 0].cpu().numpy())
    best = 1e9
    for _ in range(3):
        p.run(xs, ys)
        p.sync()
        best = min(best, p.last_kernel_ms())
    us = best * 1e3 / T
    per = 28 if opt == "adam" else 12
    byt = per * W * W * L
    print(f"C2 {opt} ({p.kernel_path}): {us:.1f} us/tick, {byt / us / 1e3:.0f} GB/s, {byt / us / 1e3 / 6560:.3f} of roofline", flush=True)
    p.close()
