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


def run_oracle_permuted(m, counts, xs, ys, lr, dtype, act_delay, learn, loss, optimizer, seed):
    """The oracle on a mathematically identical network whose hidden units are permuted
    (rows of W_l and b_l, columns of W_{l+1}): the same function, but every dot product sums
    in another order, so it is another equally valid f32 evaluation. Weights are returned in
    the original unit order."""
    import copy
    rng = np.random.default_rng(seed)
    dense = [i for i, l in enumerate(m.layers) if l.kind == "dense"]
    perms = [rng.permutation(m.layers[i].out_dim) for i in dense[:-1]]
    mp = copy.copy(m)
    mp.layers = [copy.copy(l) for l in m.layers]
    for j, i in enumerate(dense):
        W, b = np.array(m.layers[i].W), np.array(m.layers[i].b)
        if j < len(perms):
            W, b = W[perms[j]], b[perms[j]]
        if j > 0:
            W = W[:, perms[j - 1]]
        mp.layers[i].W, mp.layers[i].b = W, b
    o, l, v, Wp, bp = run_oracle(mp, counts, xs, ys, lr, dtype, act_delay, learn, loss, optimizer)
    W, bb = [], []
    for j in range(len(dense)):
        w, b = Wp[j], bp[j]
        if j < len(perms):
            inv = np.argsort(perms[j])
            w, b = w[inv], b[inv]
        if j > 0:
            w = w[:, np.argsort(perms[j - 1])]
        W.append(w)
        bb.append(b)
    return o, l, v, W, bb


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / (np.max(np.abs(b)) + 1e-30))


def frob_rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / (np.linalg.norm(b) + 1e-30))
