"""Shared test helpers: run the B200 engine and the CPU oracle on the same seeded stream."""

from __future__ import annotations

import numpy as np

from oracle import engine as oeng
from paper_2210_09147_b200 import model as mdl


def oracle_layers(m, dtype=np.float64):
    out = []
    for l in m.layers:
        if l.kind == "dense":
            out.append(("dense", np.array(l.W, dtype=dtype), np.array(l.b, dtype=dtype)))
        else:
            out.append((l.kind,))
    return out


def spec_bounds(m, counts):
    b = [0]
    for c in counts:
        b.append(b[-1] + c)
    assert b[-1] == len(m.layers)
    return b


def run_oracle(m, counts, xs, ys, lr, dtype=np.float64, act_delay=1, learn=True, loss="mse", optimizer="sgd"):
    layers = oracle_layers(m, dtype)
    p = oeng.Pipeline(layers, spec_bounds(m, counts), lr, xs[0].astype(dtype), ys[0].astype(dtype),
                      loss=loss, act_delay=act_delay, learn=learn, optimizer=optimizer)
    outs, losses, valid = [], [], []
    for t in range(len(xs)):
        o = p.step(xs[t].astype(dtype), ys[t].astype(dtype))
        outs.append(np.array(o.output, dtype=np.float64))
        losses.append(np.nan if o.loss is None else o.loss)
        valid.append(o.valid)
    W = [np.array(l[1], np.float64) for l in p.extract_weights() if l[0] == "dense"]
    b = [np.array(l[2], np.float64) for l in p.extract_weights() if l[0] == "dense"]
    return np.array(outs), np.array(losses), np.array(valid), W, b


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / (np.max(np.abs(b)) + 1e-30))


def frob_rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / (np.linalg.norm(b) + 1e-30))
