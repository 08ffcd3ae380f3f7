"""B200-native PARTIME per-tick pipeline (arXiv 2210.09147), drop-in for the reference's
`pipestream` engine API and the paper's `partime.pipeline.Pipeline`
(PAPER.md:640-672). Compute runs in libpartime_b200.so (sm_100a); see DESIGN.md."""

from . import numerics  # noqa: F401
from .model import LayerSpec, Model, StagePlan, dense, relu, tanh, mlp, init_weights  # noqa: F401
from .tensor import Tensor, as_array  # noqa: F401

__all__ = ["numerics", "Tensor", "as_array", "LayerSpec", "Model", "StagePlan", "dense", "relu", "tanh",
           "mlp", "init_weights"]
