"""Per-phase device timeline of the panel kernel (pt_set_trace): F = gather (1->3) + chunks and
publish (3->4); B = gather/delta (11->13) + chunks and publish (13->14). Usage:
python tools/panel_probe.py [width] [layers] [ticks]"""
import os
import sys
from collections import defaultdict

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2210_09147_b200 import engine, model as mdl, streams  # noqa: E402

NAMES = {1: "F.begin", 3: "F.gathered", 4: "F.end", 11: "B.begin", 13: "B.delta", 14: "B.end", 20: "tick"}


def main():
    W = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
    L = int(sys.argv[2]) if len(sys.argv) > 2 else 32
    T = int(sys.argv[3]) if len(sys.argv) > 3 else 16
    m = mdl.mlp([W] * (L + 1), seed=0)
    st = streams.SmoothStream(W, W, seed=1)
    xs, ys = st.block(0, T)
    xs, ys = xs.astype(np.float32), ys.astype(np.float32)
    opt = sys.argv[4] if len(sys.argv) > 4 else "sgd"
    p = engine.Pipeline(m, [len(m.layers)], opt, 1e-3 if opt == "sgd" else 1e-4, xs[0, 0], ys[0, 0])
    print("path", p.kernel_path)
    p.run(xs, ys)
    p.sync()
    for cta in (0, 77):
        p.set_trace(cta, 1 << 16)
        p.run(xs, ys)
        p.sync()
        ms = p.last_kernel_ms()
        cons, prod, _ = p.get_trace()
        print(f"== {L}x{W} cta {cta}: {ms * 1e3 / T:.1f} us/tick")
        dur = defaultdict(list)
        for (c0, t0), (c1, t1) in zip(cons, cons[1:]):
            dur[(c0, c1)].append(t1 - t0)
        for k in sorted(dur, key=lambda k: -sum(dur[k])):
            v = np.array(dur[k])
            print(f"  {NAMES.get(k[0], k[0]):>11} -> {NAMES.get(k[1], k[1]):<11} n={len(v):4d} median={np.median(v) / 1e3:6.2f}us"
                  f" total={v.sum() / 1e3 / T:7.1f}us/tick")
        if prod:
            pt = np.array([t for _, t in prod])
            print(f"  producer: {len(pt)} loads, median gap {np.median(np.diff(pt)) / 1e3:.2f}us")
    # all-CTA step ends (codes 4 / 14): completion spread per step
    p.set_trace(-1, 1 << 20)
    p.run(xs, ys)
    p.sync()
    import ctypes
    from paper_2210_09147_b200 import _lib
    cap = 1 << 20
    buf = np.zeros(cap, np.uint64)
    _lib.check(p._lib.pt_get_trace(p._h, buf.ctypes.data_as(ctypes.c_void_p), cap), "get_trace")
    G = 128
    nev = 2 * L * T  # F and B step ends per tick (stage-1 layer 0 B included)
    ev = buf[: (cap // G) * G].reshape(-1, G)[:nev].astype(np.int64)
    ev = ev[(ev > 0).all(axis=1)]
    spread = (ev.max(axis=1) - ev.min(axis=1)) / 1e3
    step = np.diff(ev.max(axis=1)) / 1e3
    k = 2 * L
    sF = [spread[i] for i in range(len(spread)) if (i % k) < L]
    sB = [spread[i] for i in range(len(spread)) if (i % k) >= L]
    dF = [step[i] for i in range(len(step)) if ((i + 1) % k) < L and (i + 1) % k > 0]
    dB = [step[i] for i in range(len(step)) if ((i + 1) % k) > L]
    print(f"all-CTA step ends: F spread median {np.median(sF):.2f}us, B spread median {np.median(sB):.2f}us;"
          f" step time (last-to-last) F median {np.median(dF):.2f}us, B median {np.median(dB):.2f}us")
    p.close()


if __name__ == "__main__":
    main()
