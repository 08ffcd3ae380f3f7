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
Every source is deterministic given its seed and single-driver
(SPEC.md:382).
"""

from __future__ import annotations

import math

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
