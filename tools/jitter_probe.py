"""Race detector for the tile kernel: random sleeps in every role (PT_JITTER ns) must leave
the results bitwise equal to an unperturbed run (one process, no time-slicing)."""
import os, sys, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
if len(sys.argv) > 1 and sys.argv[1] == "child":
    from paper_2210_09147_b200 import engine, model as mdl, streams
    case, out = sys.argv[2], sys.argv[3]
    mb = "mb" in case
    widths = [64, 96, 96, 96, 32] if mb else [256, 512, 512, 256, 256]
    counts = [7] if case.startswith("d1") else [4, 3]
    M, T = (4 if mb else 16), 24
    st = streams.SmoothStream(widths[0], widths[-1], seed=5, batch=M)
    xs, ys = st.block(0, T)
    p = engine.Pipeline(mdl.mlp(widths, seed=4), counts, "sgd", 0.05, xs[0], ys[0], learn=not case.endswith("inf"),
                        timeout_ms=60000)
    assert p.kernel_path == ("tick" if mb else "tile")
    if "dev" in case:
        import torch
        o, l, v = p.run(torch.from_numpy(xs.astype(np.float32)).cuda(), torch.from_numpy(ys.astype(np.float32)).cuda())
        p.sync()
        o = o.cpu().numpy()
    else:
        o, l, v = p.run(xs.astype(np.float32), ys.astype(np.float32))
    np.save(out, o)
    sys.exit(0)
for case in sys.argv[1:] or ["d1-inf", "d1", "d2", "mb-d2", "d1-mb", "mb-d2-dev", "d2-dev"]:
    subprocess.run([sys.executable, __file__, "child", case, "/tmp/ref.npy"], env=dict(os.environ, PT_JITTER="0"), check=True)
    ref = np.load("/tmp/ref.npy")
    for jit, mask in [("0", "3"), ("2000", "3"), ("8000", "3"), ("200000", "255"), ("1000000", "1023")]:
        subprocess.run([sys.executable, __file__, "child", case, "/tmp/j.npy"],
                       env=dict(os.environ, PT_JITTER=jit, PT_JITTER_MASK=mask), check=True)
        o = np.load("/tmp/j.npy")
        T = o.shape[0]
        bad = [t for t in range(T) if not np.array_equal(o[t], ref[t])]
        print(f"{case} jitter {jit} ns (1 in {int(mask) + 1}): bitwise equal {not bad} first bad tick {bad[:1]}", flush=True)
