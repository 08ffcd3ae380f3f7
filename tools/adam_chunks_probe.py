import os, sys
sys.path.insert(0, '/root/repo')
os.chdir(os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np
from paper_2210_09147_b200 import engine, model as mdl, streams
W, L, T = 2048, 32, 4
m = mdl.mlp([W] * (L + 1), seed=0)
xs, ys = streams.SmoothStream(W, W, seed=1).block(0, T)
xs, ys = xs.astype(np.float32), ys.astype(np.float32)
p = engine.Pipeline(m, [len(m.layers)], "adam", 1e-4, xs[0, 0], ys[0, 0])
p.run(xs, ys); p.sync()
p.set_trace(5, 1 << 18)
p.run(xs, ys); p.sync()
cons, prod, chunks = p.get_trace()
# take tick 2's B steps: consumer events 11 (B.begin), 13 (B.delta), 14 (B.end)
ev = sorted([(t, 'C%d' % c) for c, t in cons] + [(t, 'P%d' % c) for c, t in prod] + [(t, 'K%d' % c) for c, t in chunks])
# find the 40th B.delta
bd = [t for c, t in cons if c == 13]
t0 = bd[len(bd) // 2]
win = [(round((t - t0) / 1e3, 2), n) for t, n in ev if -5000 <= t - t0 <= 50000]
print(win[:200])
p.close()
