"""torch.nn.Sequential -> Model (dense / relu / tanh layer specs).

The paper's library expects a torch.nn.Sequential. The B200
path implements Linear, ReLU and Tanh. Any other module raises
NotImplementedError with its index.
"""

from __future__ import annotations

import numpy as np

from ..model import LayerSpec, Model


def sequential_to_model(net, loss="mse"):
    import torch.nn as nn

    layers = []
    for i, mod in enumerate(net):
        if isinstance(mod, nn.Linear):
            if mod.bias is None:
                # the kernels train every layer's bias; a zero bias would be trained and then
                # dropped by sync_to_net, so the synced net would not reproduce the pipeline
                raise NotImplementedError(f"module {i}: nn.Linear(bias=False) is not supported on the B200 "
                                          "path (every dense layer trains a bias)")
            W = mod.weight.detach().float().cpu().numpy().copy()
            b = mod.bias.detach().float().cpu().numpy().copy()
            layers.append(LayerSpec("dense", mod.in_features, mod.out_features, W=W, b=b))
        elif isinstance(mod, nn.ReLU):
            layers.append(LayerSpec("relu"))
        elif isinstance(mod, nn.Tanh):
            layers.append(LayerSpec("tanh"))
        else:
            raise NotImplementedError(f"module {i} ({type(mod).__name__}) is not supported on the B200 path "
                                      "(Linear, ReLU and Tanh are)")
    if not layers or layers[0].kind != "dense":
        raise ValueError("the network must start with a Linear layer")
    dense = [l for l in layers if l.kind == "dense"]
    return Model(layers=layers, loss=loss, input_shape=(dense[0].in_dim,), output_dim=dense[-1].out_dim)
