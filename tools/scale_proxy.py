"""Per-GPU share under one-stage-per-GPU scaling, measured on one GPU: each stage of a D-stage
plan runs alone as a D=1 pipeline of its layers (its compute without the NVLink hop, an upper
bound on the per-GPU tick rate at D GPUs). The bottleneck stage sets the pipeline's tick.
- C2 (32 x 2048): equal split, 32/N layers per GPU; at N=8 a stage's weights fit in L2.
- C5 (uneven 1024..8192, 24 layers): the DP-balanced plan of bench.balanced_counts."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import tools.configs_probe as cp

ROOF = 6560.0e9  # MEASURED_PEAKS.json hbm_gbs


def stage_time(widths, ticks=32):
    from paper_2210_09147_b200 import engine, model as mdl, streams
    m = mdl.mlp(widths, seed=0)
    st = streams.SmoothStream(widths[0], widths[-1], seed=1)
    xs, ys = st.block(0, ticks)
    xs = torch.tensor(xs, dtype=torch.float32, device="cuda")
    ys = torch.tensor(ys, dtype=torch.float32, device="cuda")
    p = engine.Pipeline(m, [len(m.layers)], "sgd", 1e-3, xs[0, 0].cpu().numpy(), ys[0, 0].cpu().numpy())
    best = 1e9
    for _ in range(3):
        p.run(xs, ys)
        p.sync()
        best = min(best, p.last_kernel_ms())
    p.close()
    return best * 1e3 / ticks


if __name__ == "__main__":
    for n in (1, 2, 4, 8):
        L = 32 // n
        cp.probe(f"C2 stage share at N={n} ({L} layers)", [2048] * (L + 1), 1, ticks=64)
    # C3 at D=8: 8 inference layers of 4096 per GPU; C4 at D=8: 4 learning layers of 4096,
    # micro-batch 16 (tile kernel)
    cp.probe("C3 stage share at N=8 (8 x 4096, inference)", [4096] * 9, 1, learn=False, ticks=32)
    cp.probe("C4 stage share at N=8 (4 x 4096, M=16)", [4096] * 5, 1, M=16, ticks=16)
    import bench
    c5 = [1024, 2048, 4096, 8192, 8192, 4096, 2048, 1024] * 3 + [1024]
    for D in (2, 4, 8):
        counts = bench.balanced_counts(c5, D, True)
        dense, b = [], 0
        for c in counts:  # dense layers per stage (dense + relu pairs, linear head)
            dense.append((c + 1) // 2)
        per, u = [], 0
        for k in dense:
            w = c5[u:u + k + 1]
            per.append((stage_time(w), bench.algorithmic_bytes_per_tick(w)))
            u += k
        worst = max(t for t, _ in per)
        byt = max(b for _, b in per)
        print(f"C5 D={D} plan {counts}: stage us/tick {[round(t, 1) for t, _ in per]}, bottleneck {worst:.1f} us "
              f"-> {1e6 / worst:.0f} samples/s (roofline of the bottleneck-bytes stage {byt / ROOF * 1e6:.1f} us)",
              flush=True)
