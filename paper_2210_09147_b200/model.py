"""Model description for the drop-in API: LayerSpec / Model / StagePlan.

Mirrors the reference types in SPEC.md:37-50 (LayerSpec, Model) and
SPEC.md:132-135 (StagePlan). Weight init follows SPEC.md:106: W and b are
uniform in +-1/sqrt(fan_in), seeded per layer from (global_seed, layer_index).

The B200 path fuses each dense layer with the activation that follows it
(dense, dense+relu, dense+tanh). Stage boundaries must not split such a pair.
conv2d, avgpool2d, flatten and residual_add are valid in the reference
 but out of scope here. All benchmark configs are MLPs
(SURVEY.md §2 row 4); building them raises NotImplementedError.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

SUPPORTED = ("dense", "relu", "tanh")
REFERENCE_ONLY = ("conv2d", "avgpool2d", "flatten", "residual_add")
# SPEC.md:74-75 names the loss "softmax_cross_entropy"; "softmax_ce" is the short form
LOSS_ALIASES = {"softmax_cross_entropy": "softmax_ce"}


def canonical_loss(name):
    return LOSS_ALIASES.get(name, name)


@dataclass
class LayerSpec:
    kind: str
    in_dim: int = 0
    out_dim: int = 0
    W: np.ndarray | None = None   # [out_dim, in_dim]
    b: np.ndarray | None = None   # [out_dim]
    init_seed: int = 0
    version: int = 0              # per-stage weight version w_h^(t) stamped by extract (Eq. 7)


@dataclass
class Model:
    layers: list
    loss: str = "mse"
    input_shape: tuple = ()
    output_dim: int = 0

    def __post_init__(self):
        self.loss = canonical_loss(self.loss)

    @property
    def dense_layers(self):
        return [l for l in self.layers if l.kind == "dense"]


@dataclass
class StagePlan:
    """Contiguous partition of the model's layers into D stages.

    boundaries: D half-open ranges [a_h, b_h) over Model.layers indices.
    """
    boundaries: list
    worker_assignment: list = field(default_factory=list)
    predicted_stage_cost: list = field(default_factory=list)

    @property
    def D(self):
        return len(self.boundaries)

    def layer_counts(self):
        """Printable layer-count form, e.g. [8, 10, 12, 11]."""
        return [b - a for a, b in self.boundaries]

    @classmethod
    def from_counts(cls, counts):
        if any(c < 1 for c in counts):
            raise ValueError(f"stage layer counts must be >= 1, got {counts}")
        bounds, a = [], 0
        for c in counts:
            bounds.append((a, a + c))
            a += c
        return cls(boundaries=bounds)

    def validate(self, n_layers):
        if self.D < 1:
            raise ValueError("a stage plan needs at least one stage")
        if self.D > n_layers:
            raise ValueError(f"D={self.D} > L={n_layers} (SPEC.md:151)")
        prev = 0
        for h, (a, b) in enumerate(self.boundaries):
            if a != prev or b <= a:
                raise ValueError(f"stage plan is not contiguous/covering at stage {h + 1}: {self.boundaries}")
            prev = b
        if prev != n_layers:
            raise ValueError(f"stage plan covers {prev} of {n_layers} layers")


def dense(in_dim, out_dim, seed=0):
    return LayerSpec("dense", in_dim, out_dim, init_seed=seed)


def relu():
    return LayerSpec("relu")


def tanh():
    return LayerSpec("tanh")


def init_weights(model: Model, seed: int = 0, dtype=np.float32):
    """U(+-1/sqrt(fan_in)) per dense layer, rng seeded with (seed, layer_index)."""
    for idx, layer in enumerate(model.layers):
        if layer.kind != "dense":
            continue
        rng = np.random.default_rng([seed, idx])
        bound = 1.0 / np.sqrt(layer.in_dim)
        W = rng.random((layer.out_dim, layer.in_dim), dtype=np.float64)
        W *= 2.0 * bound
        W -= bound
        layer.W = W.astype(dtype, copy=False)
        b = rng.random(layer.out_dim, dtype=np.float64) * (2.0 * bound) - bound
        layer.b = b.astype(dtype, copy=False)
        layer.init_seed = seed
    return model


def mlp(widths, act="relu", loss="mse", seed=0, dtype=np.float32, init=True):
    """Dense layers widths[0]->widths[1]->...; `act` after every dense layer except the
    last (linear head), as in the benchmark configs."""
    layers = []
    for i in range(len(widths) - 1):
        layers.append(dense(widths[i], widths[i + 1], seed))
        if i < len(widths) - 2 and act != "none":
            layers.append(LayerSpec(act))
    m = Model(layers=layers, loss=loss, input_shape=(widths[0],), output_dim=widths[-1])
    if init:
        init_weights(m, seed, dtype)
    return m


def fuse(model: Model):
    """Model layers -> fused units [(spec_index_of_dense, act)] and a map from SPEC layer
    index to fused unit index. Raises on layer kinds the B200 path does not implement."""
    units = []
    owner = []
    for i, layer in enumerate(model.layers):
        if layer.kind in REFERENCE_ONLY:
            raise NotImplementedError(f"layer {i} ({layer.kind}) is not implemented on the B200 path")
        if layer.kind not in SUPPORTED:
            raise ValueError(f"layer {i}: unknown layer kind {layer.kind!r}")
        if layer.kind == "dense":
            if units and layer.in_dim != model.layers[units[-1][0]].out_dim:
                raise ValueError(f"layer {i}: dense expects input {model.layers[units[-1][0]].out_dim}, "
                                 f"declared {layer.in_dim}")
            units.append([i, "none"])
        else:
            if i == 0 or model.layers[i - 1].kind != "dense":
                raise NotImplementedError(
                    f"layer {i} ({layer.kind}) does not directly follow a dense layer; only dense+activation "
                    "pairs are fused on the B200 path")
            units[-1][1] = layer.kind
        owner.append(len(units) - 1)
    if not units:
        raise ValueError("model has no dense layer")
    return [tuple(u) for u in units], owner


def plan_to_units(model: Model, plan: StagePlan, owner):
    """StagePlan over SPEC layers -> stage_first_layer over fused units (D+1 entries)."""
    plan.validate(len(model.layers))
    first = []
    for h, (a, b) in enumerate(plan.boundaries):
        if a > 0 and owner[a] == owner[a - 1]:
            raise ValueError(f"stage boundary {h}->{h + 1} splits dense layer {owner[a]} from its activation")
        first.append(owner[a])
    first.append(owner[-1] + 1)
    return first
