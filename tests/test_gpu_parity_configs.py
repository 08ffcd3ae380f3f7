"""GPU parity at the shapes bench.py quotes (BASELINE.json configs), against the f64 oracle with
the f32 oracle as calibration and a delta-W check (tests/test_gpu_parity.py::_case; bars
there). Each case runs on one GPU with the stage split bench.py uses, so every number in the
bench line's `other_configs` (and the headline C2) is backed by a parity test of the same
shape, kernel and stage count:

- C2: 32 x 2048 ReLU MLP, batch 1, learning, N = 50 ticks at D = 1, 2 and 8;
- C3: 64 x 4096 inference wave, D = 8, 16 ticks;
- C4: 32 x 4096, micro-batch 16 and 32 (tcgen05 tile kernel), D = 8, 8 ticks;
- C5: uneven widths 1024..8192 (24 layers), DP-balanced (bench.balanced_counts), D = 8, 8 ticks.

The oracle runs on the host in f64 and f32 (numpy + BLAS); the C4/C5 cases take a minute or
two of host time each.
"""

import numpy as np
import pytest

from tests.test_gpu_parity import _case

pytestmark = pytest.mark.gpu

C5 = [1024, 2048, 4096, 8192, 8192, 4096, 2048, 1024] * 3 + [1024]


def _bench_counts(widths, D, learn):
    import bench
    return bench.balanced_counts(widths, D, learn)


@pytest.mark.parametrize("D", [1, 2, 8])
def test_c2_50_ticks(D):
    """Config 2 (the headline): 32 x 2048, batch 1, SGD lr 1e-3, 50 ticks, equal stages."""
    import bench
    _case([2048] * 33, bench.plan_counts(32, D), 50, 1e-3)


def test_c2_adam_d1():
    """Config 2's shape with Adam on the panel kernel (a bench other_configs line), 12 ticks."""
    _case([2048] * 33, [63], 12, 1e-4, optimizer="adam")


def test_c3_inference_d8():
    """Config 3: 64 x 4096 inference-only forward wave, D = 8 (bench split), 16 ticks."""
    w = [4096] * 65
    _case(w, _bench_counts(w, 8, False), 16, 0.0, learn=False)


@pytest.mark.parametrize("M", [16, 32])
def test_c4_tile_d8(M):
    """Config 4: 32 x 4096, micro-batch 16 (and 32, bench's C4_m32 line) on the tcgen05 tile
    kernel, D = 8, 8 ticks."""
    from paper_2210_09147_b200 import engine, model as mdl
    w = [4096] * 33
    counts = _bench_counts(w, 8, True)
    p = engine.Pipeline(mdl.mlp(w, seed=0), counts, "sgd", 1e-3, np.zeros((M, 4096), np.float32),
                        np.zeros((M, 4096), np.float32))
    assert p.kernel_path == "tile"
    p.close()
    _case(w, counts, 8, 1e-3, M=M)


def test_c4_tile_d8_adam_ce():
    """Config 4's shape with Adam and softmax-CE on the tile kernel (a bench other_configs line)."""
    from paper_2210_09147_b200 import engine, model as mdl
    w = [4096] * 33
    counts = _bench_counts(w, 8, True)
    p = engine.Pipeline(mdl.mlp(w, seed=0, loss="softmax_ce"), counts, "adam", 1e-4,
                        np.zeros((16, 4096), np.float32), np.zeros(16, np.float32))
    assert p.kernel_path == "tile"
    p.close()
    _case(w, counts, 10, 1e-4, M=16, optimizer="adam", loss="softmax_ce")  # valid outputs from t = D - 1 = 7


@pytest.mark.parametrize("D", [2, 4, 8])
def test_c5_uneven(D):
    """Config 5: uneven widths 1024..8192, DP-balanced stages (the scale proxy's plans),
    D = 2 / 4 / 8, 2D + 2 ticks."""
    _case(C5, _bench_counts(C5, D, True), 2 * D + 2, 1e-3)
