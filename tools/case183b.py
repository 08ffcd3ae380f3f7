import sys; sys.path.insert(0, "/root/repo")
from tests.test_gpu_parity import _case


def run(tag, *a, **k):
    try:
        e = _case(*a, **k)
        print(f"{tag}: ok ({e:.1e})", flush=True)
    except AssertionError as ex:
        print(f"{tag}: FAIL {ex}", flush=True)


for W in ([66, 184, 244, 50, 279], [66, 184, 244, 279], [66, 184, 16, 279], [66, 184, 50, 279],
          [66, 300, 279], [66, 184, 184, 279], [128, 128, 128, 128], [66, 128, 128, 279]):
    L = len(W) - 1
    run(f"{W} D1 M16", W, [2 * L - 1], 13, 0.01, seed=830, M=16)
run("[128]*4 M16 relu lr0.001", [128] * 4, [5], 13, 0.001, seed=830, M=16)
run("[128]*4 M16 tanh", [128] * 4, [5], 13, 0.01, seed=830, M=16, act="tanh")
