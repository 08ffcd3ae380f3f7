"""pipestream.netcore domain types: LayerSpec, Model, seeded init.

The layer math of SPEC.md:53-88 (layer_forward / layer_backward / loss / update) runs
inside the B200 tick kernels (paper_2210_09147_b200/csrc/pt_kernels.cuh), fused per
stage and per tick; it is not exposed as separate host calls.
"""
from paper_2210_09147_b200.model import (LayerSpec, Model, canonical_loss, dense, init_weights, mlp,  # noqa: F401
                                         relu, tanh)
