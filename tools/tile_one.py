"""One tile-kernel launch (C4 shape, 8 layers, 2 ticks) for ncu."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2210_09147_b200 import engine, model as mdl, streams
L = int(sys.argv[1]) if len(sys.argv) > 1 else 8
learn = (sys.argv[2] != "infer") if len(sys.argv) > 2 else True
widths = [4096] * (L + 1)
m = mdl.mlp(widths, seed=0)
st = streams.SmoothStream(4096, 4096, seed=1, batch=16)
xs, ys = st.block(0, 2)
xs = torch.tensor(xs, dtype=torch.float32, device="cuda"); ys = torch.tensor(ys, dtype=torch.float32, device="cuda")
p = engine.Pipeline(m, [2 * L - 1], "sgd", 1e-3 if learn else 0.0, xs[0].cpu().numpy(), ys[0].cpu().numpy(), learn=learn)
assert p.kernel_path == "tile"
for _ in range(2):
    p.run(xs, ys); p.sync()
print("ms", p.last_kernel_ms())
