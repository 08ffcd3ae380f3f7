"""Chunk-level timeline of the panel kernel on one CTA (pt_set_trace): when each chunk's load
was issued by the producer (codes 40 F / 41 B), when the consumers found it ready (7 F / 8 B),
and where that falls inside the step (1/3/4 F begin/gathered/end, 11/13/14 B). Usage:
python tools/panel_chunks.py [width] [layers] [ticks] [cta]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2210_09147_b200 import engine, model as mdl, streams  # noqa: E402


def main():
    W = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
    L = int(sys.argv[2]) if len(sys.argv) > 2 else 32
    T = int(sys.argv[3]) if len(sys.argv) > 3 else 8
    cta = int(sys.argv[4]) if len(sys.argv) > 4 else 0
    m = mdl.mlp([W] * (L + 1), seed=0)
    st = streams.SmoothStream(W, W, seed=1)
    xs, ys = st.block(0, T)
    xs, ys = xs.astype(np.float32), ys.astype(np.float32)
    p = engine.Pipeline(m, [len(m.layers)], "sgd", 1e-3, xs[0, 0], ys[0, 0])
    p.run(xs, ys)
    p.sync()
    p.set_trace(cta, 1 << 18)
    p.run(xs, ys)
    p.sync()
    print(f"{L}x{W}: {p.last_kernel_ms() * 1e3 / T:.1f} us/tick")
    cons, prod, chunks = p.get_trace()
    p.close()
    t0 = cons[0][1]
    # walk the consumer steps of the middle ticks, pairing chunk events in order
    ready = {7: [t for c, t in chunks if c == 7], 8: [t for c, t in chunks if c == 8]}
    issue = {7: [t for c, t in prod if c == 40], 8: [t for c, t in prod if c == 41]}
    idx = {7: 0, 8: 0}
    stats = {"F": [], "B": []}
    step = None
    for code, t in cons:
        if code in (1, 11):
            step = ("F" if code == 1 else "B", t)
        elif code in (3, 13):
            step = step + (t,)
        elif code in (4, 14) and step is not None and len(step) == 3:
            kind, tb, tg = step
            k = 7 if kind == "F" else 8
            rs, iss = [], []
            while idx[k] < len(ready[k]) and ready[k][idx[k]] <= t:
                rs.append(ready[k][idx[k]])
                iss.append(issue[k][idx[k]] if idx[k] < len(issue[k]) else np.nan)
                idx[k] += 1
            if rs:
                stats[kind].append((tg - tb, [r - tg for r in rs], [r - i for r, i in zip(rs, iss)],
                                    [tb - i for i in iss], t - rs[-1]))
    # dot phase: ready (7) -> dot done (9) per chunk, and the reduction barrier (10)
    ev = [(c, t) for c, t in chunks if c in (7, 9, 10)]
    d9, d10 = [], []
    for (c0, t0), (c1, t1) in zip(ev, ev[1:]):
        if c1 == 9:
            d9.append(t1 - t0)
        if c1 == 10 and c0 == 9:
            d10.append(t1 - t0)
    if d9:
        print(f"dot: median gap before each dot-done {np.median(d9) / 1e3:.2f}us; last dot -> reduction barrier {np.median(d10) / 1e3:.2f}us")
    for kind in ("F", "B"):
        v = stats[kind][len(stats[kind]) // 4:]
        if not v:
            continue
        gw = np.median([x[0] for x in v]) / 1e3
        rr = np.median(np.array([x[1] for x in v if len(x[1]) == len(v[0][1])]), axis=0) / 1e3
        lat = np.median(np.array([x[2] for x in v if len(x[2]) == len(v[0][2])]), axis=0) / 1e3
        ahead = np.median(np.array([x[3] for x in v if len(x[3]) == len(v[0][3])]), axis=0) / 1e3
        tail = np.median([x[4] for x in v]) / 1e3
        print(f"{kind}: gather {gw:.2f}us; chunk ready after gathered {np.round(rr, 2)}us; issue->ready "
              f"{np.round(lat, 2)}us; issued before step begin {np.round(ahead, 2)}us; last ready->end {tail:.2f}us")


if __name__ == "__main__":
    main()
