"""Narrow down a randomised-parity failure (generic tick path, micro-batch 16)."""
import sys; sys.path.insert(0, "/root/repo")
from tests.test_gpu_parity import _case


def run(tag, *a, **k):
    try:
        e = _case(*a, **k)
        print(f"{tag}: ok ({e:.1e})", flush=True)
    except AssertionError as ex:
        print(f"{tag}: FAIL {ex}", flush=True)


W = [66, 184, 244, 50, 16, 279]
run("base M16", W, [2, 7], 13, 0.01, seed=830, M=16)
run("M8", W, [2, 7], 13, 0.01, seed=830, M=8)
run("M12", W, [2, 7], 13, 0.01, seed=830, M=12)
run("D1 M16", W, [9], 13, 0.01, seed=830, M=16)
run("seed1 M16", W, [2, 7], 13, 0.01, seed=1, M=16)
run("lr0.001 M16", W, [2, 7], 13, 0.001, seed=830, M=16)
run("T6 M16", W, [2, 7], 6, 0.01, seed=830, M=16)
run("short net M16", [66, 184, 279], [2, 1], 13, 0.01, seed=830, M=16)
run("w64 M16", [64, 184, 244, 50, 16, 279], [2, 7], 13, 0.01, seed=830, M=16)
run("grid 16 M16", W, [2, 7], 13, 0.01, seed=830, M=16, grid=16)
