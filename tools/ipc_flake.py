"""Two-process (CUDA IPC) D=2 runs on one GPU vs the single-process pipeline, repeated, to
localise intermittent mismatches. Env: FLAKE_N trials, FLAKE_M batch, FLAKE_LEARN 0/1,
FLAKE_LR, FLAKE_T ticks."""
import os, sys, socket
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch.multiprocessing as mp

M = int(os.environ.get("FLAKE_M", "4"))
LEARN = os.environ.get("FLAKE_LEARN", "1") == "1"
LR = float(os.environ.get("FLAKE_LR", "0.05"))
T = int(os.environ.get("FLAKE_T", "16"))
WIDTHS, COUNTS = [64, 96, 96, 96, 32], [4, 3]


def data():
    from paper_2210_09147_b200 import streams
    st = streams.SmoothStream(WIDTHS[0], WIDTHS[-1], seed=5, batch=M)
    xs, ys = st.block(0, T)
    return xs.astype(np.float32), ys.astype(np.float32)


def s0(a):
    return a[0] if M > 1 else a[0, 0]


def worker(rank, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE="2")
    import torch
    import torch.distributed as dist
    from paper_2210_09147_b200 import dist as pdist, model as mdl
    dist.init_process_group("gloo", rank=rank, world_size=2)
    torch.cuda.set_device(0)
    xs, ys = data()
    pipe = pdist.build_distributed(mdl.mlp(WIDTHS, seed=4), COUNTS, "sgd", LR, s0(xs), s0(ys), timeout_ms=60000,
                                   learn=LEARN)
    first = pipe.local_first == 0
    outs, losses, valid = pipe.run(torch.from_numpy(xs).cuda() if first else None,
                                   None if first else torch.from_numpy(ys).cuda(), T)
    pipe.sync()
    res = {"rank": rank, "weights": [pipe.get_layer(j)[0] for j in pipe._local_units()]}
    if not first:
        res["outs"] = outs.cpu().numpy()
    q.put(res)
    dist.barrier()
    pipe.close()
    dist.destroy_process_group()


def main():
    from paper_2210_09147_b200 import engine, model as mdl
    xs, ys = data()
    ref = engine.Pipeline(mdl.mlp(WIDTHS, seed=4), COUNTS, "sgd", LR, s0(xs), s0(ys), learn=LEARN)
    o, _, _ = ref.run(xs, ys)
    W = [ref.get_layer(j)[0] for j in range(ref.L)]
    ref.close()
    ctx = mp.get_context("spawn")
    for trial in range(int(os.environ.get("FLAKE_N", "8"))):
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]
        q = ctx.Queue()
        procs = [ctx.Process(target=worker, args=(r, port, q)) for r in range(2)]
        for p in procs: p.start()
        got = {}
        for _ in procs:
            r = q.get(timeout=300); got[r["rank"]] = r
        for p in procs: p.join(timeout=120)
        go, ro = got[1]["outs"].reshape(T, M, -1), o.reshape(T, M, -1)
        bad = [t for t in range(T) if not np.array_equal(go[t], ro[t])]
        mine = got[0]["weights"] + got[1]["weights"]
        wbad = [j for j in range(len(W)) if not np.array_equal(mine[j], W[j])]
        if bad:
            t0 = bad[0]
            rows = [m for m in range(M) if not np.array_equal(go[t0, m], ro[t0, m])]
            print(f"M={M} learn={LEARN} lr={LR} trial {trial}: MISMATCH first tick {t0} rows {rows} "
                  f"max {np.abs(go[t0] - ro[t0]).max():.3g} weights {wbad}", flush=True)
        else:
            print(f"M={M} learn={LEARN} lr={LR} trial {trial}: equal, weights differ {wbad}", flush=True)


if __name__ == "__main__":
    main()
