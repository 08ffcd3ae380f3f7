"""streams: drift2d, DatasetFile round trip and validation, replay window mechanics."""

import math

import numpy as np
import pytest

from paper_2210_09147_b200 import streams


def test_replay_window_examples(tmp_path):
    # W=3 over a,b,c,d: [a,a,a] -> [b,a,a] -> [c,b,a] -> [d,c,b]
    x = np.arange(4, dtype=np.float32)[:, None] * np.ones((4, 2), np.float32)
    p = tmp_path / "d.bin"
    streams.dataset_write(p, x, np.arange(4))
    r = streams.ReplayStream(streams.dataset_read(p), 3)
    got = [list(lab) for _, lab, _ in r]
    assert got == [[0, 0, 0], [1, 0, 0], [2, 1, 0], [3, 2, 1]]
    with pytest.raises(StopIteration):
        next(r)
    xs, ys = streams.ReplayStream(streams.dataset_read(p), 3, passes=2).block(3, 3)
    assert ys.tolist() == [[3, 2, 1], [0, 3, 2], [1, 0, 3]]
    assert np.array_equal(xs[:, :, 0], ys)


def test_replay_errors(tmp_path):
    p = tmp_path / "e.bin"
    streams.dataset_write(p, np.zeros((0, 3), np.float32), np.zeros(0, np.int32))
    ds = streams.dataset_read(p)
    assert ds.n == 0
    with pytest.raises(ValueError, match="empty"):
        next(streams.ReplayStream(ds, 2))
    with pytest.raises(ValueError):
        streams.ReplayStream(ds, 0)


def test_dataset_round_trip_and_truncation(tmp_path):
    rng = np.random.default_rng(0)
    x = rng.standard_normal((7, 3, 4)).astype(np.float32)
    lab = rng.integers(0, 10, (7, 2)).astype(np.int32)
    p = tmp_path / "r.bin"
    streams.dataset_write(p, x, lab)
    ds = streams.dataset_read(p)
    assert ds.shape == (3, 4) and np.array_equal(ds.x, x) and np.array_equal(ds.labels, lab)
    data = p.read_bytes()
    (tmp_path / "t.bin").write_bytes(data[:-5])
    with pytest.raises(ValueError, match=f"expected {len(data)} bytes .* got {len(data) - 5}"):
        streams.dataset_read(tmp_path / "t.bin")


def test_drift2d_smooth_and_seeded():
    s = streams.Drift2dStream(n_classes=3, rho=0.01, sigma=0.1, seed=4, radius=2.0)
    for t in (0, 5, 100):
        step = np.linalg.norm(s.means(t + 1) - s.means(t), axis=1)
        assert np.all(step <= 0.01 * 2.0 + 1e-12)  # the chord is at most the arc rho R
        assert np.allclose(step, 2 * 2.0 * math.sin(0.01 / 2))
    a = [next(s) for _ in range(5)]
    b = [next(streams.Drift2dStream(3, 0.01, 0.1, 4, 2.0)) for _ in range(1)]
    assert np.array_equal(a[0][0], b[0][0]) and a[0][1] == b[0][1]
    # rho = 0: stationary means
    z = streams.Drift2dStream(2, 0.0, 0.1, 1)
    assert np.array_equal(z.means(0), z.means(1000))
    with pytest.raises(ValueError):
        streams.Drift2dStream(2, -1.0)
    xs, ys = streams.Drift2dStream(2, 0.0, 0.1, 1, batch=3).block(0, 4)
    assert xs.shape == (4, 3, 2) and ys.shape == (4, 3) and ys[0, 1] == ys[0, 0]
