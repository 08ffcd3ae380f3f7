"""Do persistent tick kernels of two processes time-sliced on one GPU stay bitwise equal to a
solo run? Each process runs its own single-process pipeline (no IPC). Variants localise a
timing-dependent result: TS_CASE = d2 (D=2 learning), d1 (D=1 learning), inf (D=2 inference),
lr0 (D=2, lr=0), tile / tile1 (tcgen05 tile kernel, micro-batch 16, D=2 / D=1), mb / mb1
(tick kernel, micro-batch 4, D=2 / D=1); a -inf or -lr0
suffix applies to any case."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch.multiprocessing as mp

T = int(os.environ.get("TS_TICKS", "200"))


def job(rank, q, case):
    import torch
    from paper_2210_09147_b200 import engine, model as mdl, streams
    torch.cuda.set_device(0)
    tile = case.startswith("tile")
    mb = case.startswith("mb")
    widths = [256, 512, 512, 256, 256] if tile else [64, 96, 96, 96, 32] if mb else [32, 64, 64, 64, 16]
    M = 16 if tile else 4 if mb else 1
    m = mdl.mlp(widths, seed=4)
    st = streams.SmoothStream(widths[0], widths[-1], seed=5, batch=M)
    xs, ys = st.block(0, T)
    counts = [7] if case.split("-")[0] in ("d1", "tile1", "mb1") else [4, 3]
    lr = 0.0 if case.endswith("lr0") else 0.05
    s0 = (lambda a: a[0]) if M > 1 else (lambda a: a[0, 0])
    p = engine.Pipeline(m, counts, "sgd", lr, s0(xs), s0(ys), timeout_ms=60000, learn=not case.endswith("inf"))
    xs_d = torch.from_numpy(xs.astype(np.float32)).cuda(); ys_d = torch.from_numpy(ys.astype(np.float32)).cuda()
    o, l, v = p.run(xs_d, ys_d)
    p.sync()
    W = [p.get_layer(j)[0] for j in range(p.L)]
    q.put((rank, o.cpu().numpy(), W))
    p.close()


if __name__ == "__main__":
    ctx = mp.get_context("spawn")
    cases = sys.argv[1:] or ["d2", "d1", "inf", "lr0"]
    for case in cases:
        for trial in range(int(os.environ.get("TS_TRIALS", "3"))):
            q = ctx.Queue()
            ps = [ctx.Process(target=job, args=(r, q, case)) for r in range(2)]
            for p in ps: p.start()
            res = {r: (o, W) for r, o, W in (q.get(timeout=300) for _ in ps)}
            for p in ps: p.join()
            q = ctx.Queue(); solo = ctx.Process(target=job, args=(9, q, case)); solo.start()
            _, ref, Wref = q.get(timeout=300); solo.join()
            for r in (0, 1):
                o, W = res[r]
                bad = np.nonzero(~np.all(o.reshape(T, -1) == ref.reshape(T, -1), axis=1))[0]
                wbad = [j for j in range(len(W)) if not np.array_equal(W[j], Wref[j])]
                print(f"{case} trial {trial} proc{r}: outputs equal {bad.size == 0} "
                      f"(first differing tick {bad[0] if bad.size else '-'}), weights differ in layers {wbad}", flush=True)
