"""CPU reference scaling: the oracle pipeline on C2 with D worker threads and
two barriers per tick, each worker's BLAS limited to floor(cores / D) threads,
a bounded sample per D. Usage: cpu_scaling.py [seconds per D]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from threadpoolctl import threadpool_limits

import bench
from oracle import engine as oeng
from paper_2210_09147_b200 import model as mdl, streams

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 10.0
cores = len(os.sched_getaffinity(0))
widths = [2048] * 33
m = mdl.mlp(widths, seed=0, dtype=np.float32)
layers = [("dense", l.W, l.b) if l.kind == "dense" else (l.kind,) for l in m.layers]
xs, ys = streams.SmoothStream(2048, 2048, seed=1).block(0, 64)
xs, ys = xs.astype(np.float32), ys.astype(np.float32)
base = None
for D in (1, 2, 4, 8):
    counts = bench.plan_counts(32, D)
    bounds = [0]
    for c in counts:
        bounds.append(bounds[-1] + c)
    with threadpool_limits(max(1, cores // D)):
        p = oeng.Pipeline(layers, bounds, 1e-3, xs[0], ys[0], threads=D > 1)
        for t in range(2 * D):  # warm-up 2D ticks
            p.step(xs[t % 64], ys[t % 64])
        t0, n = time.perf_counter(), 0
        while time.perf_counter() - t0 < budget:
            p.step(xs[n % 64], ys[n % 64])
            n += 1
        el = time.perf_counter() - t0
        p.close()
    rate = n / el
    base = base or rate
    print(f"C2 CPU D={D}: {rate:.2f} samples/s ({n} ticks in {el:.1f}s, {cores} cores, "
          f"{max(1, cores // D)} BLAS threads per worker), speed-up {rate / base:.2f}", flush=True)
