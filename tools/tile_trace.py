"""Per-phase device timeline of the tcgen05 tile kernel (CTA 0, SIMT thread 0)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from collections import defaultdict
from paper_2210_09147_b200 import engine, model as mdl, streams

NAMES = {1: "compute.begin", 2: "compute.end", 3: "barrier1", 4: "finalize", 5: "barrier2", 6: "chunk.begin",
         7: "full.seen", 11: "mdone.j-2", 12: "opnd.rdy", 13: "lopass.end", 22: "mma.hi.issued", 23: "mma.prep.seen", 8: "prep.done", 8: "grpB.wait", 9: "grpB.mdone", 10: "grpB.done", 14: "update.math", 20: "mma.prep", 21: "mma.commit",
         30: "tma.issue"}

def run(widths, counts, ticks=2, M=16, learn=True, cta=0, opt="sgd"):
    m = mdl.mlp(widths, seed=0)
    st = streams.SmoothStream(widths[0], widths[-1], seed=1, batch=M)
    xs, ys = st.block(0, ticks)
    xs = torch.tensor(xs, dtype=torch.float32, device="cuda"); ys = torch.tensor(ys, dtype=torch.float32, device="cuda")
    p = engine.Pipeline(m, counts, opt, (1e-3 if opt == "sgd" else 1e-4) if learn else 0.0, xs[0].cpu().numpy(), ys[0].cpu().numpy(), learn=learn)
    assert p.kernel_path == "tile", p.kernel_path
    p.run(xs, ys); p.sync()
    p.set_trace(cta, 1 << 14)
    p.run(xs, ys); p.sync()
    ms = p.last_kernel_ms()
    import ctypes
    from paper_2210_09147_b200 import _lib as L_
    cap = p._trace_cap
    buf = np.zeros(cap, np.uint64)
    L_.check(p._lib.pt_get_trace(p._h, buf.ctypes.data_as(ctypes.c_void_p), cap), "get_trace")
    dec = lambda a: [(int(v >> np.uint64(56)), int(v & np.uint64(0x00FFFFFFFFFFFFFF))) for v in a if v]
    q4 = cap // 4
    cons, grpb, mma, prod = dec(buf[:q4]), dec(buf[q4:2 * q4]), dec(buf[2 * q4:3 * q4]), dec(buf[3 * q4:])
    if grpb:
        d = defaultdict(list)
        for (c0, t0), (c1, t1) in zip(grpb, grpb[1:]):
            d[(c0, c1)].append(t1 - t0)
        for k in sorted(d, key=lambda k: -sum(d[k])):
            v = np.array(d[k])
            print(f"  group B {NAMES.get(k[0], k[0]):>12} -> {NAMES.get(k[1], k[1]):<12} n={len(v):4d} median={np.median(v) / 1e3:6.2f}us total={v.sum() / 1e3 / ticks:8.1f}us/tick")
    L = len(widths) - 1
    print(f"== {widths[0]}x{L} M={M} {opt} learn={learn} counts={counts}: {ms * 1e3 / ticks:.1f} us/tick")
    dur = defaultdict(list)
    for (c0, t0), (c1, t1) in zip(cons, cons[1:]):
        dur[(c0, c1)].append(t1 - t0)
    for k in sorted(dur, key=lambda k: -sum(dur[k])):
        v = np.array(dur[k])
        print(f"  {NAMES.get(k[0], k[0]):>14} -> {NAMES.get(k[1], k[1]):<14} n={len(v):4d} median={np.median(v) / 1e3:8.2f}us "
              f"total={v.sum() / 1e3 / ticks:9.1f}us/tick")
    if mma:
        t = np.array([x for _, x in mma])
        codes = [c for c, _ in mma]
        issue = [t[i + 1] - t[i] for i in range(len(t) - 1) if codes[i] == 20 and codes[i + 1] == 21]
        gap = [t[i + 1] - t[i] for i in range(len(t) - 1) if codes[i] == 21 and codes[i + 1] == 20]
        print(f"  mma: issue (prep->commit) median {np.median(issue) / 1e3:.2f}us; commit->next prep median {np.median(gap) / 1e3:.2f}us")
        d = defaultdict(list)
        for i in range(len(t) - 1):
            d[(codes[i], codes[i + 1])].append(t[i + 1] - t[i])
        for k in sorted(d):
            print(f"    mma {NAMES.get(k[0], k[0])} -> {NAMES.get(k[1], k[1])}: median {np.median(d[k]) / 1e3:.2f}us n={len(d[k])}")
    if prod:
        t = np.array([x for _, x in prod])
        print(f"  producer: {len(t)} loads, median gap {np.median(np.diff(t)) / 1e3:.2f}us")
        fs = [x for c_, x in cons if c_ == 7]
        n = min(len(fs), len(t))
        lat = np.array(fs[:n]) - t[:n]
        print(f"  TMA issue -> group A sees full: median {np.median(lat) / 1e3:.2f}us p10 {np.percentile(lat, 10) / 1e3:.2f} p90 {np.percentile(lat, 90) / 1e3:.2f}")
        mp = [x for c_, x in mma if c_ == 20]
        n2 = min(len(mp), len(t))
        lat2 = np.array(mp[:n2]) - t[:n2]
        print(f"  TMA issue -> MMA starts chunk: median {np.median(lat2) / 1e3:.2f}us")
    base = cons[0][1]
    print("  first SIMT events:", [(NAMES.get(c, c), round((x - base) / 1e3, 2)) for c, x in cons[:60]])
    p.close()

if __name__ == "__main__":
    if len(sys.argv) > 1:  # optimizer (sgd / adam), micro-batch
        run([4096] * 9, [15], ticks=2, opt=sys.argv[1], M=int(sys.argv[2]) if len(sys.argv) > 2 else 16)
    else:
        run([4096] * 9, [15], ticks=2, learn=False)
        run([4096] * 9, [15], ticks=2)
