"""Repeat the tile-kernel determinism case (D=2, micro-batch 16, 256-512 widths) many times:
unsplit runs and runs split over two calls, each compared bitwise with the first unsplit run.
Reports how often and where they differ."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2210_09147_b200 import engine, model as mdl, streams

widths, counts, M, T = [256, 512, 512, 256], [2, 3], 16, 8
st = streams.SmoothStream(widths[0], widths[-1], seed=1, batch=M)
xs, ys = st.block(0, T)
xs, ys = xs.astype(np.float32), ys.astype(np.float32)


def one(split, learn=True):
    p = engine.Pipeline(mdl.mlp(widths, seed=0), counts, "sgd", 0.02, xs[0], ys[0], learn=learn)
    assert p.kernel_path == "tile"
    if split:
        parts = [p.run(xs[i:j], ys[i:j]) for i, j in ((0, 3), (3, 8))]
        o = np.concatenate([q[0] for q in parts])
    else:
        o = p.run(xs, ys)[0]
    W = [p.get_layer(j)[0] for j in range(p.L)]
    p.close()
    return o, W


if __name__ == "__main__":
    n = int(os.environ.get("DET_N", "20"))
    for learn in (True, False):
        ref, Wr = one(False, learn)
        for split in (False, True):
            bad = []
            for k in range(n):
                o, W = one(split, learn)
                d = [t for t in range(T) if not np.array_equal(o[t], ref[t])]
                wd = [j for j in range(len(W)) if not np.array_equal(W[j], Wr[j])]
                if d or wd:
                    rows = [m for m in range(M) if d and not np.array_equal(o[d[0], m], ref[d[0], m])]
                    bad.append((k, d[:3], rows[:6], wd))
            print(f"learn={learn} split={split}: {len(bad)}/{n} differ {bad[:4]}", flush=True)
