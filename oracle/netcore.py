"""netcore oracle: layer forward/backward, losses, optimizers, sequential step.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py). This restates SPEC.md:26-121.
Layers are plain tuples so that the oracle has no dependency on the product:
  ("dense", W[out,in], b[out])   y = x @ W.T + b        (Eq. 1)
  ("relu",)                       y = max(0, x)
  ("tanh",)                       y = tanh(x)
Activations carry a leading batch axis [M, n]; M=1 is the
per-sample stream case.
"""

from __future__ import annotations

import numpy as np

try:  # in-place rank-k update for the f32 CPU baseline; numpy path otherwise
    from scipy.linalg import blas as _blas
except Exception:  # pragma: no cover
    _blas = None


# --------------------------------------------------------------------------
# layer_forward / layer_backward
# --------------------------------------------------------------------------

def layer_forward(layer, x):
    """SPEC.md:53-61. Pure; x is [M, n_in]."""
    kind = layer[0]
    if kind == "dense":
        W, b = layer[1], layer[2]
        if x.shape[-1] != W.shape[1]:
            raise ValueError(f"dense expects input dim {W.shape[1]}, got {x.shape[-1]}")
        return x @ W.T + b
    if kind == "relu":
        return np.maximum(x, 0)
    if kind == "tanh":
        return np.tanh(x)
    raise ValueError(f"unsupported layer kind {kind!r}")


def layer_backward(layer, x, upstream):
    """returns (input_grad, weight_grads or None).

    dense: dW = upstream^T x (outer product at M=1), db = sum_M upstream,
    input_grad = upstream @ W (the pre-update W, Eq. 9-10).
    relu: gate on sign, input_grad = upstream * [x > 0].
    tanh: input_grad = upstream * (1 - tanh(x)^2).
    """
    kind = layer[0]
    if kind == "dense":
        W = layer[1]
        if upstream.shape[-1] != W.shape[0]:
            raise ValueError(f"dense backward expects upstream dim {W.shape[0]}, got {upstream.shape[-1]}")
        gin = upstream @ W
        return gin, DenseGrad(upstream, x)
    if kind == "relu":
        return upstream * (x > 0), None
    if kind == "tanh":
        t = np.tanh(x)
        return upstream * (1 - t * t), None
    raise ValueError(f"unsupported layer kind {kind!r}")


class DenseGrad:
    """GradientBundle entry of a dense layer: dW = upstream^T x, db = sum_M upstream.

    dW is materialised on first access, so an SGD step can apply the same
    rank-M update in place through BLAS without allocating [out, in].
    """

    __slots__ = ("upstream", "x", "_dW")

    def __init__(self, upstream, x):
        self.upstream, self.x, self._dW = upstream, x, None

    @property
    def dW(self):
        if self._dW is None:
            self._dW = self.upstream.T @ self.x
        return self._dW

    @property
    def db(self):
        return self.upstream.sum(axis=0)

    def __getitem__(self, i):  # (dW, db) tuple view
        return (self.dW, self.db)[i]

    def __iter__(self):
        return iter((self.dW, self.db))


# --------------------------------------------------------------------------
# losses
# --------------------------------------------------------------------------

def loss_eval(kind, out, target):
    """mse = mean over all M*F elements; softmax_ce = mean over M of -log softmax[target]."""
    if kind == "mse":
        d = out - target
        return float(np.mean(d * d))
    if kind == "softmax_ce":
        t = np.asarray(target).astype(np.int64).reshape(-1)
        if np.any(t < 0) or np.any(t >= out.shape[-1]):
            raise ValueError("cross-entropy target out of class range")
        p = softmax(out)
        return float(-np.mean(np.log(p[np.arange(out.shape[0]), t])))
    raise ValueError(f"unknown loss {kind!r}")


def loss_grad(kind, out, target):
    """dL/d(out). mse: 2(o-y)/(M*F). softmax_ce: (softmax - onehot)/M."""
    if kind == "mse":
        return 2.0 * (out - target) / out.size
    if kind == "softmax_ce":
        t = np.asarray(target).astype(np.int64).reshape(-1)
        if np.any(t < 0) or np.any(t >= out.shape[-1]):
            raise ValueError("cross-entropy target out of class range")
        g = softmax(out)
        g[np.arange(out.shape[0]), t] -= 1
        return g / out.shape[0]
    raise ValueError(f"unknown loss {kind!r}")


def softmax(z):
    z = z - z.max(axis=-1, keepdims=True)
    e = np.exp(z)
    return e / e.sum(axis=-1, keepdims=True)


# --------------------------------------------------------------------------
# optimizers
# --------------------------------------------------------------------------

class SGD:
    """Plain SGD, w -= lr * grad, applied in place."""

    def __init__(self, lr):
        self.lr = lr

    def apply(self, layer, grad):
        W, b = layer[1], layer[2]
        lr = self.lr
        if lr == 0:
            return  # lr = 0 leaves weights bit-identical
        if grad._dW is None and _blas is not None and W.flags.c_contiguous \
                and W.dtype in (np.float32, np.float64):
            # W -= lr * upstream^T x, in place through BLAS ger/gemm on W^T (F-order view).
            x, up = grad.x, grad.upstream
            ger = _blas.sger if W.dtype == np.float32 else _blas.dger
            gemm = _blas.sgemm if W.dtype == np.float32 else _blas.dgemm
            if up.shape[0] == 1:
                ger(-lr, x[0], up[0], a=W.T, overwrite_a=1)
            else:
                gemm(-lr, x.T, up, beta=1.0, c=W.T, overwrite_c=1)
        else:
            W -= lr * grad.dW
        b -= lr * grad.db


class Adam:
    """Adam (beta1=0.9, beta2=0.999, eps=1e-8); state lives with its weights."""

    def __init__(self, lr, betas=(0.9, 0.999), eps=1e-8):
        self.lr, self.b1, self.b2, self.eps = lr, betas[0], betas[1], eps
        self.state = {}

    def apply(self, layer, grads):
        key = id(layer[1])
        st = self.state.setdefault(key, [0, [np.zeros_like(layer[1]), np.zeros_like(layer[2])],
                                         [np.zeros_like(layer[1]), np.zeros_like(layer[2])]])
        st[0] += 1
        step = st[0]
        for p, g, m, v in zip((layer[1], layer[2]), grads, st[1], st[2]):
            m *= self.b1
            m += (1 - self.b1) * g
            v *= self.b2
            v += (1 - self.b2) * g * g
            mh = m / (1 - self.b1 ** step)
            vh = v / (1 - self.b2 ** step)
            p -= self.lr * mh / (np.sqrt(vh) + self.eps)


def make_optimizer(kind, lr):
    if kind == "sgd":
        return SGD(lr)
    if kind == "adam":
        return Adam(lr)
    raise ValueError(f"unknown optimizer {kind!r}")


# --------------------------------------------------------------------------
# block forward/backward helpers shared by sequential_step and the engine
# --------------------------------------------------------------------------

def block_forward(layers, x):
    """Forward through a list of layers; returns (out, inputs) where inputs[j]
    is the input of layer j (the activation cache of SPEC.md:196, 256)."""
    inputs = []
    a = x
    for layer in layers:
        inputs.append(a)
        a = layer_forward(layer, a)
    return a, inputs


def block_backward(layers, inputs, g):
    """Reverse pass with the given cache (pre-update weights); returns (input_grad, per-layer grads)."""
    grads = [None] * len(layers)
    for j in range(len(layers) - 1, -1, -1):
        g, grads[j] = layer_backward(layers[j], inputs[j], g)
    return g, grads


def apply_updates(layers, grads, opt):
    for j, layer in enumerate(layers):
        if grads[j] is not None:
            opt.apply(layer, grads[j])


def sequential_step(layers, x, target, lr=None, optimizer=None, loss="mse", step_index=0):
    """full forward, full backward, single in-place update.

    Returns (output, loss, grads). Non-finite loss raises with the step index.
    """
    opt = optimizer if optimizer is not None else SGD(lr)
    out, inputs = block_forward(layers, x)
    lval = loss_eval(loss, out, target)
    if not np.isfinite(lval):
        raise FloatingPointError(f"non-finite loss at step {step_index}")
    g = loss_grad(loss, out, target)
    _, grads = block_backward(layers, inputs, g)
    apply_updates(layers, grads, opt)
    return out, lval, grads


def forward_only(layers, x):
    return block_forward(layers, x)[0]
