"""C2 tick time with and without the weight write-back (PT_DBG bit 4): the upper bound of
what deferring the write-back (lazy rank-k updates) could save."""
import os, sys, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 1 and sys.argv[1] == "child":
    import numpy as np, torch
    from paper_2210_09147_b200 import engine, model as mdl, streams
    widths = [2048] * 33
    m = mdl.mlp(widths, seed=0)
    st = streams.SmoothStream(2048, 2048, seed=1)
    xs, ys = st.block(0, 64)
    xs = torch.tensor(xs, dtype=torch.float32, device="cuda"); ys = torch.tensor(ys, dtype=torch.float32, device="cuda")
    p = engine.Pipeline(m, [len(m.layers)], "sgd", 1e-3, xs[0, 0].cpu().numpy(), ys[0, 0].cpu().numpy())
    best = 1e9
    for r in range(5):
        p.run(xs, ys); p.sync()
        if r: best = min(best, p.last_kernel_ms())
    print(f"PT_DBG={os.environ.get('PT_DBG','0')} {sys.argv[2:]}: {best * 1e3 / 64:.1f} us/tick")
    if len(sys.argv) > 2 and sys.argv[2] == "trace":
        import tools.trace_probe as tp
        tp.run(widths, 1)
    sys.exit(0)
for dbg in ["0", "16", "24"]:
    env = dict(os.environ, PT_DBG=dbg)
    subprocess.run([sys.executable, __file__, "child"] + (["trace"] if dbg == "16" else []), env=env)
