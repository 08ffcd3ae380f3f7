"""Repeat the two-process IPC run and report where it diverges from one process."""
import os, socket, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from tests.test_gpu_ipc import _worker
import torch.multiprocessing as mp
from paper_2210_09147_b200 import engine, model as mdl, streams

def once():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]
    ctx = mp.get_context("spawn"); q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(2)]
    for p in procs: p.start()
    got = {}
    for _ in procs:
        r = q.get(timeout=300); got[r["rank"]] = r
    for p in procs: p.join(timeout=120)
    m = mdl.mlp([32, 64, 64, 64, 16], seed=4)
    st = streams.SmoothStream(32, 16, seed=5)
    xs, ys = st.block(0, 12)
    ref = engine.Pipeline(m, [4, 3], "sgd", 0.05, xs[0, 0], ys[0, 0])
    o, l, v = ref.run(xs.astype(np.float32), ys.astype(np.float32))
    bad = [t for t in range(12) if not np.array_equal(got[1]["outs"][t], o[t])]
    W = [ref.get_layer(j) for j in range(ref.L)]
    wb = [j for j, ((a, _), (b, _)) in enumerate(zip(got[0]["weights"] + got[1]["weights"], W)) if not np.array_equal(a, b)]
    print("first bad tick", bad[:3], "bad layers", wb, flush=True)

if __name__ == "__main__":
    for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 6):
        once()
