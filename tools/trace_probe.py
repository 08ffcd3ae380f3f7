"""Per-phase device timeline of one CTA (diagnostics via pt_set_trace)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from collections import defaultdict
from paper_2210_09147_b200 import engine, model as mdl, streams

NAMES = {1: "F.begin", 2: "F.credit", 3: "F.input", 4: "F.chunks", 5: "F.end",
         11: "B.begin", 12: "B.act", 13: "B.delta", 14: "B.chunks", 15: "B.push", 20: "tick"}

def run(widths, D, learn=True, ticks=8, cta=0):
    m = mdl.mlp(widths, seed=0)
    L = len(widths) - 1
    per = [L // D + (1 if i < L % D else 0) for i in range(D)]
    counts, u = [], 0
    for c in per:
        counts.append(sum(2 if (u + j) < L - 1 else 1 for j in range(c))); u += c
    st = streams.SmoothStream(widths[0], widths[-1], seed=1)
    xs, ys = st.block(0, ticks)
    xs = torch.tensor(xs, dtype=torch.float32, device="cuda"); ys = torch.tensor(ys, dtype=torch.float32, device="cuda")
    p = engine.Pipeline(m, counts, "sgd", 1e-3, xs[0, 0].cpu().numpy(), ys[0, 0].cpu().numpy(), learn=learn)
    p.run(xs, ys); p.sync()
    p.set_trace(cta, 1 << 16)
    p.run(xs, ys); p.sync()
    ms = p.last_kernel_ms()
    cons, prod, chunks = p.get_trace()
    print(f"== widths {widths[0]}x{L} D={D} learn={learn} cta={cta}: {ms*1e3/ticks:.1f} us/tick")
    # phase durations: consecutive events
    dur = defaultdict(list)
    for (c0, t0), (c1, t1) in zip(cons, cons[1:]):
        dur[(c0, c1)].append(t1 - t0)
    for k in sorted(dur, key=lambda k: -sum(dur[k])):
        v = np.array(dur[k])
        print(f"  {NAMES.get(k[0],k[0]):>12} -> {NAMES.get(k[1],k[1]):<12} n={len(v):4d} median={np.median(v)/1e3:7.2f}us "
              f"total={v.sum()/1e3/ticks:8.1f}us/tick")
    if prod:
        pt = np.array([t for _, t in prod])
        gaps = np.diff(pt)
        print(f"  producer: {len(pt)} loads, median gap {np.median(gaps)/1e3:.2f}us, p90 {np.percentile(gaps,90)/1e3:.2f}us")
    if prod and chunks:
        n = min(len(prod), len(chunks))
        lat = np.array([chunks[i][1] - prod[i][1] for i in range(n)])
        print(f"  chunk issue->consumer-ready: median {np.median(lat)/1e3:.2f}us p10 {np.percentile(lat,10)/1e3:.2f} p90 {np.percentile(lat,90)/1e3:.2f}us")
        ct = np.array([t for _, t in chunks[:n]])
        fwd = [i for i in range(1, n) if chunks[i][0] == 6]
        print(f"  consumer inter-chunk gap (fwd) median {np.median(np.diff(ct)[[i-1 for i in fwd]])/1e3:.2f}us")
        rec = np.array([prod[i][1] - chunks[i - 5][1] for i in range(5, n)])
        print(f"  slot recycle (ready[c-5] -> issue[c]): median {np.median(rec)/1e3:.2f}us p90 {np.percentile(rec,90)/1e3:.2f}us")
    if chunks:
        bw = [(chunks[i + 1][1] - chunks[i][1]) for i in range(len(chunks) - 1) if chunks[i][0] == 8 and chunks[i + 1][0] == 7]
        if bw:
            bw = np.array(bw)
            print(f"  backward chunk data wait: median {np.median(bw)/1e3:.2f}us p90 {np.percentile(bw,90)/1e3:.2f}us, "
                  f"total {bw.sum()/1e3/ticks:.1f}us/tick over {len(bw)//ticks} chunks/tick")
        b7 = [chunks[i][1] for i in range(len(chunks)) if chunks[i][0] == 7]
        b8 = [chunks[i][1] for i in range(len(chunks)) if chunks[i][0] == 8]
    # a snippet of the raw timeline around tick 4
    base = cons[0][1]
    print("  first 40 events:", [(NAMES.get(c, c), round((t - base) / 1e3, 2)) for c, t in cons[:40]])
    p.close()

if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    if which == "small":
        run([2048] * 5, 1, ticks=16)
        run([2048] * 5, 1, ticks=16, learn=False)
        sys.exit(0)
    run([2048] * 33, 1)
    if which == "all":
        run([2048] * 33, 1, cta=100)
        run([2048] * 33, 1, learn=False)
        run([2048] * 33, 8)
