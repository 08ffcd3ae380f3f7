"""Tile handles created and destroyed in sequence with other allocations in between (as in a
long test session): the last handle's results must equal a fresh run of the same case.
A stale TMA descriptor-cache entry for a reused tensor-map address would point the copies at
another handle's (freed) weights. PT_LIBNAME selects the build under test."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2210_09147_b200 import engine, model as mdl, streams


def case(widths, seed, T=6):
    M = 16
    st = streams.SmoothStream(widths[0], widths[-1], seed=seed, batch=M)
    xs, ys = st.block(0, T)
    xs, ys = xs.astype(np.float32), ys.astype(np.float32)
    p = engine.Pipeline(mdl.mlp(widths, seed=seed), [len(widths) * 2 - 3], "sgd", 0.02, xs[0], ys[0])
    assert p.kernel_path == "tile"
    o = p.run(xs, ys)[0]
    p.close()
    return o


if __name__ == "__main__":
    shapes = [[256, 512, 512, 256], [512, 256, 256], [256, 256, 512, 512, 256], [768, 512, 256]]
    refs = {i: case(s, i) for i, s in enumerate(shapes)}
    bad = 0
    junk = []
    rng = np.random.default_rng(0)
    for trial in range(int(os.environ.get("REUSE_N", "40"))):
        junk.append(torch.empty(int(rng.integers(1, 64)) << 16, device="cuda"))
        if len(junk) > 6:
            junk.pop(int(rng.integers(len(junk))))
        i = int(rng.integers(len(shapes)))
        o = case(shapes[i], i)
        if not np.array_equal(o, refs[i]):
            bad += 1
            print(f"trial {trial} shape {i}: MISMATCH max {np.abs(o - refs[i]).max():.3g}", flush=True)
    print(f"{os.environ.get('PT_LIBNAME', 'libpartime_b200.so')}: {bad} mismatches", flush=True)
