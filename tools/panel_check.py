"""Quick GPU check of the batch-1 panel kernel: panel vs f64 oracle (and vs the tick kernel)
on a few seeded cases; prints the errors and the kernel path. Usage: python tools/panel_check.py"""

import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2210_09147_b200 import engine, model as mdl, streams  # noqa: E402
from tests.helpers import frob_rel, rel, run_oracle  # noqa: E402

CASES = [
    # widths, counts, T, lr, act, act_delay, loss, grid
    ([5, 7, 6, 3], [5], 30, 0.05, "relu", 1, "mse", 0),
    ([5, 7, 6, 3], [2, 3], 30, 0.05, "relu", 1, "mse", 0),
    ([6, 9, 8, 4], [2, 3], 30, 0.05, "tanh", 1, "mse", 0),
    ([16, 24, 24, 8], [2, 3], 40, 0.05, "relu", 0, "mse", 0),
    ([40, 130, 70, 9], [2, 3], 25, 0.05, "relu", 1, "mse", 3),
    ([64, 96, 96, 32], [2, 3], 20, 0.05, "relu", 1, "softmax_ce", 0),
    ([64, 96, 96, 32], [5], 20, 0.05, "relu", 1, "softmax_ce", 0),
    ([512] * 9, [8, 7], 60, 1e-3, "relu", 1, "mse", 0),
    ([2048] * 5, [7], 12, 1e-3, "relu", 1, "mse", 0),
    ([1024, 4096, 1024, 2048], [5], 10, 1e-3, "relu", 1, "mse", 0),
]


def one(widths, counts, T, lr, act, act_delay, loss, grid, panel=True):
    os.environ["PT_PANEL"] = "1" if panel else "0"
    m = mdl.mlp(widths, act=act, seed=0, loss=loss)
    st = streams.SmoothStream(widths[0], widths[-1], seed=1)
    xs, ys = st.block(0, T)
    if loss == "softmax_ce":
        ys = np.argmax(ys, axis=-1).astype(np.float64)
    W0 = [l.W.astype(np.float64) for l in m.dense_layers]
    pipe = engine.Pipeline(m, counts, "sgd", lr, xs[0, 0], ys[0, 0], act_delay=act_delay, grid=grid)
    path = pipe.kernel_path
    t0 = time.time()
    outs, losses, valid = pipe.run(xs.astype(np.float32), ys.astype(np.float32))
    dt = time.time() - t0
    got = pipe.extract_weights()
    pipe.close()
    return path, dt, outs, losses, valid, got, W0, (m, counts, xs, ys, lr, act_delay, loss)


def main():
    bad = 0
    for c in CASES:
        path, dt, outs, losses, valid, got, W0, (m, counts, xs, ys, lr, ad, loss) = one(*c)
        o64, l64, v64, W64, b64 = run_oracle(m, counts, xs, ys, lr, np.float64, ad, True, loss)
        vm = v64
        e_out = rel(outs.reshape(o64.shape), o64)
        e_loss = rel(losses[vm], l64[vm]) if vm.any() else 0.0
        o32, l32, v32, W32, b32 = run_oracle(m, counts, xs, ys, lr, np.float32, ad, True, loss)
        e_dw = 0.0
        e_b = 0.0
        per = []
        for j, l in enumerate(got.dense_layers):
            dW64 = W64[j] - W0[j]
            if np.linalg.norm(dW64) > 0:
                e = frob_rel(l.W.astype(np.float64) - W0[j], dW64)
                e32 = frob_rel(W32[j] - W0[j], dW64)
                per.append(f"{e:.1e}/{e32:.1e}")
                e_dw = max(e_dw, e / max(1.0, e32 / 2.5e-4))
            e_b = max(e_b, frob_rel(l.b, b64[j]))
        print("   per-layer dW err (gpu/f32 oracle):", " ".join(per))
        print("   out err per tick:", " ".join(f"{rel(outs[t].reshape(o64[t].shape), o64[t]):.0e}" for t in range(0, len(o64), max(1, len(o64) // 12))))
        ok = e_out < 1e-4 and e_loss < 1e-4 and e_dw < 1e-3 and e_b < 1e-4 and np.array_equal(valid.astype(bool), v64)
        bad += not ok
        print(f"{'OK ' if ok else 'BAD'} {path:5s} {str(c[0][:6]):28s} D={len(c[1])} {c[4]} ad={c[5]} {c[6]:10s} "
              f"out {e_out:.2e} loss {e_loss:.2e} dW {e_dw:.2e} b {e_b:.2e}  ({dt:.2f}s)", flush=True)
        # bit-level comparison with the tick kernel (different summation order: tolerance only)
        p2 = one(*c, panel=False)
        print(f"    vs tick: out {rel(outs, p2[2]):.2e}; tick vs oracle out {rel(p2[2].reshape(o64.shape), o64):.2e}", flush=True)
    print("bad cases:", bad)


if __name__ == "__main__":
    main()
