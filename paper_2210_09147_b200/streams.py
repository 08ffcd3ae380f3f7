"""Stream sources (reference `streams` module).

- ConstantStream: every call returns the same (x, gamma).
- SmoothStream: the d-dimensional smooth-drift stream that every benchmark
  config uses (generalising drift2d). It is
    x_t = cos(rho t) u  + sin(rho t) v  + sigma eps_t
    y_t = cos(rho t + phi) u' + sin(rho t + phi) v'
  with u, v, u', v' ~ N(0, I) drawn from default_rng(seed), rho = 2 pi / 1000,
  sigma = 0.01, phi = 0.5, and eps_t drawn from default_rng([seed, 1, t]).
  The stream is generated in f64 and cast by the caller. With batch M > 1,
  each tick emits the sliding window [s_t, s_{t-1}, ..., s_{t-M+1}] of the
  last M samples; the cold start is filled with sample 0 (SPEC.md:358, 363,
  378).
- Drift2dStream: 2-d points from class-conditional Gaussians whose means sit
  on a circle of radius R and rotate by rho radians per step (SPEC.md:358,
  372); the label is the class index (softmax-CE target).
- DatasetFile + dataset_write / dataset_read: the SPEC's binary dataset
  format.
- ReplayStream: the sliding-window "replay batch" of PAPER §5.D over a
  DatasetFile: the window is filled with the first
  sample, then each step admits the next sample and drops the oldest; rows
  are newest first; the stream ends after `passes` sweeps.
Every source is deterministic given its seed and single-driver
(SPEC.md:382).
"""

from __future__ import annotations

import math
import struct
from dataclasses import dataclass

import numpy as np


class ConstantStream:
    def __init__(self, x, y):
        self.x, self.y, self.t = np.asarray(x), np.asarray(y), 0

    def __iter__(self):
        return self

    def __next__(self):
        t = self.t
        self.t += 1
        return self.x, self.y, t

    def block(self, t0, n):
        xs = np.broadcast_to(self.x, (n,) + self.x.shape).copy()
        ys = np.broadcast_to(self.y, (n,) + self.y.shape).copy()
        return xs, ys


class SmoothStream:
    def __init__(self, d_in, d_out, seed=0, batch=1, rho=2 * math.pi / 1000, sigma=0.01, phi=0.5):
        rng = np.random.default_rng(seed)
        self.u, self.v = rng.standard_normal(d_in), rng.standard_normal(d_in)
        self.u2, self.v2 = rng.standard_normal(d_out), rng.standard_normal(d_out)
        self.d_in, self.d_out, self.seed, self.M = d_in, d_out, seed, batch
        self.rho, self.sigma, self.phi = rho, sigma, phi
        self.t = 0

    def samples(self, t0, n):
        """Single samples s_t, t in [t0, t0+n) (t < 0 clamps to 0): x [n, d_in], y [n, d_out] f64."""
        ts = np.maximum(np.arange(t0, t0 + n), 0)
        c, s = np.cos(self.rho * ts)[:, None], np.sin(self.rho * ts)[:, None]
        x = c * self.u + s * self.v
        for i, t in enumerate(ts):
            x[i] += self.sigma * np.random.default_rng([self.seed, 1, int(t)]).standard_normal(self.d_in)
        c2 = np.cos(self.rho * ts + self.phi)[:, None]
        s2 = np.sin(self.rho * ts + self.phi)[:, None]
        y = c2 * self.u2 + s2 * self.v2
        return x, y

    def block(self, t0, n, dtype=np.float64):
        """Ticks [t0, t0+n) as arrays xs [n, M, d_in], ys [n, M, d_out]."""
        M = self.M
        x, y = self.samples(t0 - (M - 1), n + M - 1)
        xs = np.empty((n, M, self.d_in), dtype=dtype)
        ys = np.empty((n, M, self.d_out), dtype=dtype)
        for m in range(M):  # row m holds sample t-m (newest first)
            xs[:, m] = x[M - 1 - m:M - 1 - m + n]
            ys[:, m] = y[M - 1 - m:M - 1 - m + n]
        return xs, ys

    def __iter__(self):
        return self

    def __next__(self):
        xs, ys = self.block(self.t, 1)
        t = self.t
        self.t += 1
        return xs[0], ys[0], t


class Drift2dStream:
    """class k's mean at step t is R (cos(theta_k + rho t), sin(theta_k + rho t)),
    theta_k = 2 pi k / K; the class of step t and the noise are drawn from default_rng([seed, 2, t])."""

    def __init__(self, n_classes=2, rho=2 * math.pi / 1000, sigma=0.1, seed=0, radius=1.0, batch=1):
        if rho < 0:
            raise ValueError("drift2d: rho must be >= 0 (SPEC.md:349)")
        if n_classes < 1:
            raise ValueError("drift2d: n_classes must be >= 1")
        self.K, self.rho, self.sigma, self.seed, self.R, self.M = n_classes, rho, sigma, seed, radius, batch
        self.t = 0

    def means(self, t):
        """Class means at step t, [K, 2] (exposed for the drift-smoothness property)."""
        th = 2 * math.pi * np.arange(self.K) / self.K + self.rho * t
        return self.R * np.stack([np.cos(th), np.sin(th)], axis=1)

    def sample(self, t):
        t = max(int(t), 0)
        rng = np.random.default_rng([self.seed, 2, t])
        k = int(rng.integers(self.K))
        return self.means(t)[k] + self.sigma * rng.standard_normal(2), k

    def block(self, t0, n, dtype=np.float64):
        """Ticks [t0, t0+n): xs [n, M, 2], ys [n, M] class indices (newest row first)."""
        xs = np.empty((n, self.M, 2), dtype=dtype)
        ys = np.empty((n, self.M), dtype=dtype)
        for i in range(n):
            for m in range(self.M):
                xs[i, m], ys[i, m] = self.sample(t0 + i - m)
        return xs, ys

    def __iter__(self):
        return self

    def __next__(self):
        x, k = self.sample(self.t)
        t = self.t
        self.t += 1
        return x, k, t


@dataclass
class DatasetFile:
    """SPEC.md:352-355. x: [N, *shape] float32; labels: [N, arity] int32."""
    x: np.ndarray
    labels: np.ndarray

    @property
    def n(self):
        return int(self.x.shape[0])

    @property
    def shape(self):
        return tuple(self.x.shape[1:])


# header: u64 N | u32 rank | u32 dims[rank] | u32 label_arity; then N records of
# prod(dims) little-endian f32 followed by label_arity little-endian i32
def _header(n, shape, arity):
    return struct.pack(f"<QI{len(shape)}II", n, len(shape), *shape, arity)


def dataset_write(path, x, labels):
    x = np.ascontiguousarray(x, dtype="<f4")
    labels = np.asarray(labels)
    if labels.ndim == 1:
        labels = labels[:, None]
    labels = np.ascontiguousarray(labels, dtype="<i4")
    if x.ndim < 2 or labels.shape[0] != x.shape[0]:
        raise ValueError(f"dataset_write: {x.shape[0] if x.ndim else 0} samples vs {labels.shape[0]} labels")
    n, shape, arity = x.shape[0], x.shape[1:], labels.shape[1]
    feat = int(np.prod(shape))
    rec = np.empty((n, feat * 4 + arity * 4), np.uint8)
    rec[:, :feat * 4] = x.reshape(n, feat).view(np.uint8)
    rec[:, feat * 4:] = labels.view(np.uint8)
    with open(path, "wb") as f:
        f.write(_header(n, shape, arity))
        f.write(rec.tobytes())


def dataset_read(path) -> DatasetFile:
    with open(path, "rb") as f:
        data = f.read()
    if len(data) < 12:
        raise ValueError(f"dataset_read: header truncated ({len(data)} bytes)")
    n, rank = struct.unpack_from("<QI", data, 0)
    hb = 12 + 4 * rank + 4
    if len(data) < hb:
        raise ValueError(f"dataset_read: header truncated: expected {hb} bytes, got {len(data)}")
    shape = struct.unpack_from(f"<{rank}I", data, 12)
    (arity,) = struct.unpack_from("<I", data, 12 + 4 * rank)
    feat = int(np.prod(shape)) if rank else 1
    rb = 4 * feat + 4 * arity
    want = hb + n * rb
    if len(data) != want:
        raise ValueError(f"dataset_read: expected {want} bytes for {n} records, got {len(data)}")
    rec = np.frombuffer(data, np.uint8, offset=hb).reshape(n, rb)
    x = rec[:, :4 * feat].copy().view("<f4").reshape((n,) + tuple(shape)).astype(np.float32)
    labels = rec[:, 4 * feat:].copy().view("<i4").reshape(n, arity).astype(np.int32)
    return DatasetFile(x, labels)


class ReplayStream:
    """Sliding-window replay over a DatasetFile (PAPER §5.D).

    Step i admits sample i mod N (pass i // N); the window holds the W most recent
    admissions, newest first, initially W copies of sample 0. next() returns
    (x_window [W, d], label_window [W] (or [W, arity]), sample_id)."""

    def __init__(self, ds: DatasetFile, W, passes=1):
        if W < 1:
            raise ValueError("replay: W must be >= 1 (SPEC.md:349)")
        self.ds, self.W, self.passes = ds, int(W), int(passes)
        self.t = 0

    def __len__(self):
        return self.ds.n * self.passes

    def _lab(self, idx):
        lab = self.ds.labels[idx]
        return lab[..., 0] if self.ds.labels.shape[1] == 1 else lab

    def window(self, t):
        """Dataset indices in the window after admitting step t (newest first)."""
        if self.ds.n == 0:
            raise ValueError("replay over an empty dataset (N=0)")
        steps = np.maximum(t - np.arange(self.W), 0)
        return steps % self.ds.n

    def block(self, t0, n, dtype=np.float64):
        """Steps [t0, t0+n): xs [n, W, d], ys [n, W] labels. Raises past the end of the stream."""
        if t0 + n > len(self):
            raise ValueError(f"replay: steps {t0}..{t0 + n - 1} past the end ({len(self)} steps)")
        idx = np.stack([self.window(t) for t in range(t0, t0 + n)])  # [n, W]
        xs = self.ds.x.reshape(self.ds.n, -1)[idx].astype(dtype)
        return xs, self._lab(idx).astype(dtype)

    def __iter__(self):
        return self

    def __next__(self):
        if self.ds.n == 0:
            raise ValueError("replay over an empty dataset (N=0)")
        if self.t >= len(self):
            raise StopIteration
        idx = self.window(self.t)
        t = self.t
        self.t += 1
        return self.ds.x.reshape(self.ds.n, -1)[idx], self._lab(idx), t
