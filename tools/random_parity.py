"""Randomised parity sweep against the f64 oracle: random widths (1..300), depth, stage split,
activation, act_delay, batch (1, 2, 4, 16), optimizer, loss and learning rate. Uses the same
self-calibrated tolerance as tests/test_gpu_parity.py. Prints every failing case."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from tests.test_gpu_parity import _case


WMAX = int(os.environ.get("WMAX", "300"))


def random_case(rng, wmax=None):
    wmax = wmax or WMAX
    L = int(rng.integers(1, int(os.environ.get("LMAX", "5")) + 1))
    widths = [int(rng.integers(1, wmax)) for _ in range(L + 1)]
    M = int(rng.choice([1, 1, 2, 4, 16] + ([32, 64] if os.environ.get("BIG_M") else [])))
    if os.environ.get("TILE_ONLY"):
        M = 16
        widths = [256 * int(rng.integers(1, 17)) for _ in range(L + 1)]  # the tile kernel, up to 4096
    elif M == 16 and rng.random() < 0.5:
        widths = [256 * int(rng.integers(1, 3)) for _ in range(L + 1)]  # the tile kernel
    elif rng.random() < 0.3:
        widths = [int(rng.integers(1, wmax))] * (L + 1)  # uniform: concurrent local stages
    n_layers = 2 * L - 1  # dense + act pairs, linear head
    D = int(rng.integers(1, min(L, int(os.environ.get("DMAX", "4"))) + 1))
    cuts = sorted(rng.choice(np.arange(1, L), D - 1, replace=False).tolist()) if D > 1 else []
    units = np.diff([0] + cuts + [L]).tolist()
    counts, u = [], 0
    for c in units:
        counts.append(sum(2 if (u + j) < L - 1 else 1 for j in range(c)))
        u += c
    assert sum(counts) == n_layers
    loss = "softmax_ce" if rng.random() < 0.3 and widths[-1] >= 2 else "mse"
    c = dict(widths=widths, counts=counts, T=int(rng.integers(2 * D + 2, 24)), lr=float(rng.choice([0.0, 0.01, 0.05])),
                act=str(rng.choice(["relu", "tanh"])), act_delay=int(rng.integers(0, 2)), M=M,
                optimizer=str(rng.choice(["sgd", "sgd", "adam"])), loss=loss, seed=int(rng.integers(0, 1000)),
                learn=bool(rng.random() >= float(os.environ.get("P_INFER", "0"))))
    if os.environ.get("OPT"):  # e.g. OPT=adam LR=0.05: the Adam cases at the largest lr
        c["optimizer"] = os.environ["OPT"]
    if os.environ.get("LR"):
        c["lr"] = float(os.environ["LR"])
    return c


if __name__ == "__main__":
    rng = np.random.default_rng(int(os.environ.get("SEED", "0")))  # WMAX=4096: large shapes
    n, bad = int(os.environ.get("N", "40")), 0
    for k in range(n):
        c = random_case(rng)
        try:
            _case(c["widths"], c["counts"], c["T"], c["lr"], act=c["act"], seed=c["seed"], act_delay=c["act_delay"],
                  M=c["M"], optimizer=c["optimizer"], loss=c["loss"], learn=c["learn"])
        except Exception as e:  # noqa: BLE001
            bad += 1
            print(f"case {k} FAILED {c}: {type(e).__name__}: {str(e)[:200]}", flush=True)
    print(f"{bad} / {n} failed", flush=True)
