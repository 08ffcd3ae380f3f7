"""Do persistent tick kernels of two processes time-sliced on one GPU stay bitwise equal to a
solo run? Each process runs its own single-process D=2 pipeline (no IPC)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch.multiprocessing as mp

T = int(os.environ.get("TS_TICKS", "200"))

def job(rank, q):
    import torch
    from paper_2210_09147_b200 import engine, model as mdl, streams
    torch.cuda.set_device(0)
    m = mdl.mlp([32, 64, 64, 64, 16], seed=4)
    st = streams.SmoothStream(32, 16, seed=5)
    xs, ys = st.block(0, T)
    p = engine.Pipeline(m, [4, 3], "sgd", 0.05, xs[0, 0], ys[0, 0], timeout_ms=60000)
    xs_d = torch.from_numpy(xs.astype(np.float32)).cuda(); ys_d = torch.from_numpy(ys.astype(np.float32)).cuda()
    o, l, v = p.run(xs_d, ys_d)
    p.sync()
    q.put((rank, o.cpu().numpy()))
    p.close()

if __name__ == "__main__":
    ctx = mp.get_context("spawn")
    for trial in range(4):
        q = ctx.Queue()
        ps = [ctx.Process(target=job, args=(r, q)) for r in range(2)]
        for p in ps: p.start()
        res = dict(q.get(timeout=300) for _ in ps)
        for p in ps: p.join()
        q = ctx.Queue(); solo = ctx.Process(target=job, args=(9, q)); solo.start(); _, ref = q.get(timeout=300); solo.join()
        print("trial", trial, "proc0 == solo:", np.array_equal(res[0], ref), "proc1 == solo:", np.array_equal(res[1], ref), flush=True)
