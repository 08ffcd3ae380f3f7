"""Worker of tests/test_gpu_jitter.py, run in a subprocess with PT_LIBNAME pointing at
libpartime_b200_jitter.so (the engine with the PT_JITTER race detector compiled in).
Exit status 0 iff every jittered run is bitwise equal to the unperturbed one."""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_2210_09147_b200 import engine, model as mdl, streams  # noqa: E402

CASES = {"tile": ([256, 512, 512, 256, 256], 16), "tick": ([32, 64, 64, 64, 16], 1),
         "panel": ([32, 64, 64, 64, 16], 1), "panel_wide": ([256, 512, 512, 512, 128], 1),
         "panel_adam": ([256, 512, 512, 512, 128], 1), "tile_adam": ([256, 512, 512, 256, 256], 16),
         "tile_m32": ([256, 512, 512, 256, 256], 32), "tile_m32_adam": ([256, 512, 512, 256, 256], 32),
         "tile_m64": ([256, 512, 512, 256, 256], 64), "tile_m64_adam": ([256, 512, 512, 256, 256], 64),
         "tick_mb": ([64, 96, 96, 96, 32], 4), "tick_conc": ([256] * 9, 1), "tick_conc_mb": ([128] * 9, 4),
         "tick_mb_wide": ([1218, 3805, 2590, 1500], 2)}


def main(kind, counts, learn):
    widths, M = CASES[kind]
    if kind.startswith("tick"):
        os.environ["PT_PANEL"] = "0"  # the row-owned tick kernel (batch 1 defaults to the panel kernel)
    T = 16
    st = streams.SmoothStream(widths[0], widths[-1], seed=5, batch=M)
    xs, ys = st.block(0, T)
    xs, ys = xs.astype(np.float32), ys.astype(np.float32)
    s0 = (lambda a: a[0]) if M > 1 else (lambda a: a[0, 0])

    def run():
        opt = "adam" if kind.endswith("_adam") else "sgd"
        p = engine.Pipeline(mdl.mlp(widths, seed=4), counts, opt, 0.05 if opt == "sgd" else 1e-3, s0(xs), s0(ys),
                            learn=learn)
        assert p.kernel_path == kind.split("_")[0], p.kernel_path
        o, l, _ = p.run(xs, ys)
        W = [p.get_layer(j)[0] for j in range(p.L)]
        p.close()
        return o, l, W

    os.environ["PT_JITTER"] = "0"
    o0, l0, W0 = run()
    for jit, mask in (("8000", "3"), ("300000", "511")):
        os.environ["PT_JITTER"], os.environ["PT_JITTER_MASK"] = jit, mask
        o, l, W = run()
        ok = np.array_equal(o, o0) and np.array_equal(l, l0, equal_nan=True)
        ok = ok and all(np.array_equal(a, b) for a, b in zip(W, W0))
        print(f"{kind} counts={counts} learn={learn} jitter={jit}ns/1in{int(mask) + 1}: bitwise {ok}", flush=True)
        if not ok:
            return 1
    return 0


if __name__ == "__main__":
    sys.exit(main(sys.argv[1], [int(c) for c in sys.argv[2].split(",")], sys.argv[3] == "1"))
