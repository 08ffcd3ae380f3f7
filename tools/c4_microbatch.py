"""C4 network (32 x 4096, D = 8 on one GPU) on the tile kernel at micro-batches 16 / 32 / 64,
SGD and Adam: device time per tick and the HBM roofline fraction (bench.py other_configs arithmetic)."""
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import bench
from paper_2210_09147_b200 import engine, model as mdl, streams
Ms = [int(a) for a in sys.argv[1].split(",")] if len(sys.argv) > 1 else [16, 32, 64]
OPTS = sys.argv[2].split(",") if len(sys.argv) > 2 else ["sgd", "adam"]
for M in Ms:
    for opt in OPTS:
        w = [4096]*33
        m = mdl.mlp(w, seed=0, dtype=np.float32)
        st = streams.SmoothStream(4096, 4096, seed=1, batch=M)
        xs, ys = st.block(0, 8)
        xs = torch.tensor(xs, device="cuda"); ys = torch.tensor(ys, device="cuda")
        p = engine.Pipeline(m, bench.balanced_counts(w, 8, True), opt, 1e-3 if opt=="sgd" else 1e-4, xs[0].cpu().numpy(), ys[0].cpu().numpy())
        for _ in range(2):  # 16 ticks: every stage past its warm-up gate (t >= 2D - h - 1)
            p.run(xs, ys)
        best = 1e30
        for _ in range(3):
            p.run(xs, ys); p.sync(); best = min(best, p.last_kernel_ms())
        us = best*1e3/8
        byt = bench.algorithmic_bytes_per_tick(w, True, opt)
        print(f"C4 M={M} {opt} path={p.kernel_path} tick {us:.1f} us samples/s {M*1e6/us:.0f} frac {byt/(us*1e-6)/1e9/6560:.3f}", flush=True)
        p.close()
