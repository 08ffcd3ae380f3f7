#!/bin/bash
# Ring-slot / L2-prefetch sweep of the panel kernel's Adam instantiation on C2 (32 x 2048, D=1).
for nslot in 6 5 4; do
  for pf in 8 4 16; do
    echo -n "adam nslot=$nslot pf=$pf: "
    PT_NSLOT=$nslot PT_PF_CHUNKS=$pf timeout 120 python -c "
import sys; sys.path.insert(0, '.')
import numpy as np, torch
from paper_2210_09147_b200 import engine, model as mdl, streams
w = [2048] * 33
st = streams.SmoothStream(2048, 2048, seed=1)
xs, ys = st.block(0, 32)
xs = torch.tensor(xs, device='cuda'); ys = torch.tensor(ys, device='cuda')
p = engine.Pipeline(mdl.mlp(w, seed=0, dtype=np.float32), [63], 'adam', 1e-4, xs[0, 0].cpu().numpy(), ys[0, 0].cpu().numpy())
best = 1e9
for _ in range(3):
    p.run(xs, ys); p.sync(); best = min(best, p.last_kernel_ms())
print(f'{best * 1e3 / 32:.1f} us/tick')" 2>&1 | tail -1
  done
done
