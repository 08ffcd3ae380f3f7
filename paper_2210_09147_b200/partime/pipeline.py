"""partime.pipeline.Pipeline: the paper's wrapper around an nn.Sequential.

    pipeline = Pipeline(net, sample_input, balance, devices, cuda_graph, loss_fn,
                        sample_target, optim_settings)
    for idx, (inp, target) in enumerate(stream):
        pipeline.forward(inp, target)
        if idx < len(pipeline.stages) - 1: continue     # warm-up
        outputs, loss = pipeline.outputs_buffer, pipeline.loss_buffer

Each forward() is one PARTIME tick (Alg. 1), executed by the
persistent B200 tick kernel. The device-resident loop of pipeline_run replaces
the paper's CUDA Graph capture. `cuda_graph` is accepted for signature
compatibility and ignored.
"""

from __future__ import annotations

from dataclasses import dataclass

from ..engine import Pipeline as _Engine, device_map
from ..model import StagePlan
from .convert import sequential_to_model


@dataclass
class Stage:
    index: int
    modules: list
    device: object


class Pipeline:
    def __init__(self, net, sample_input, balance, devices, cuda_graph=True, loss_fn=None,
                 sample_target=None, optim_settings=None, act_delay=1):
        import torch

        loss = "mse"
        if loss_fn is not None:
            if isinstance(loss_fn, torch.nn.CrossEntropyLoss):
                loss = "softmax_ce"  # targets: class indices
                if getattr(loss_fn, "label_smoothing", 0.0) or loss_fn.weight is not None \
                        or loss_fn.ignore_index >= 0 and loss_fn.ignore_index != -100:
                    raise NotImplementedError("CrossEntropyLoss options other than the defaults are not implemented")
            elif not isinstance(loss_fn, torch.nn.MSELoss):
                raise NotImplementedError("only torch.nn.MSELoss and torch.nn.CrossEntropyLoss are implemented "
                                          "on the B200 path")
            if getattr(loss_fn, "reduction", "mean") != "mean":
                raise NotImplementedError("the loss must use reduction='mean' (SPEC.md:74)")
        lr, opt = 1e-3, "sgd"
        if optim_settings is not None:
            cls, hp = optim_settings
            if cls is torch.optim.SGD:
                extra = {k: v for k, v in hp.items() if k not in ("lr",) and v not in (0, 0.0, False, None)}
                if extra:
                    raise NotImplementedError(f"SGD options {sorted(extra)} are not implemented on the B200 path")
            elif cls is torch.optim.Adam:
                opt = "adam"  # beta = (0.9, 0.999), eps = 1e-8
                betas = tuple(hp.get("betas", (0.9, 0.999)))
                bad = {k for k, v in hp.items() if k not in ("lr", "betas", "eps") and v not in (0, 0.0, False, None)}
                if betas != (0.9, 0.999) or float(hp.get("eps", 1e-8)) != 1e-8 or bad:
                    raise NotImplementedError("Adam runs with betas=(0.9, 0.999), eps=1e-8 and no other options")
            else:
                raise NotImplementedError(f"optimizer {cls.__name__} is not implemented on the B200 path")
            lr = float(hp.get("lr", lr))
        devs = [torch.device(d) for d in devices] if devices else [torch.device("cuda", torch.cuda.current_device())]
        devs = [torch.device("cuda", d.index if d.index is not None else torch.cuda.current_device())
                if d.type == "cuda" else d for d in devs]
        # stage -> device: one device per stage, or fewer devices each taking a contiguous block
        # of stages; several devices are driven from this process by one handle
        # (peer access, NVLink peer stores between neighbouring stages)
        dmap = device_map(devs, len(balance))
        self.devices = devs
        self.net = net
        model = sequential_to_model(net)
        model.loss = loss
        plan = StagePlan.from_counts(list(balance))
        si = sample_input.detach().cpu().numpy() if hasattr(sample_input, "detach") else sample_input
        st = sample_target.detach().cpu().numpy() if hasattr(sample_target, "detach") else sample_target
        self._eng = _Engine(model, plan, opt, lr, si, st, act_delay=act_delay, devices=dmap)
        # physical devices of the stages (the engine reports them; PT_VIRTUAL_DEVICES may fold
        # the requested ordinals onto fewer GPUs)
        phys = self._eng.stage_devices
        self.device = torch.device("cuda", phys[len(balance)])  # outputs_buffer / loss_buffer: with stage D
        self.input_device = torch.device("cuda", phys[1])
        mods = list(net)
        self.stages, a = [], 0
        for h, c in enumerate(balance):
            self.stages.append(Stage(h, mods[a:a + c], torch.device("cuda", phys[h + 1])))
            a += c
        shape = (self._eng.F,) if self._eng._squeeze else (self._eng.M, self._eng.F)
        self.outputs_buffer = torch.zeros(shape, device=self.device)
        self.loss_buffer = torch.zeros((), device=self.device)
        self.cuda_graph = cuda_graph

    def forward(self, inp, target=None):
        """One tick: forward, push, delayed backward and update on every stage (Alg. 1)."""
        import torch

        inp = inp.to(self.input_device) if hasattr(inp, "to") else torch.as_tensor(inp, device=self.input_device)
        if target is not None:
            target = target.to(self.device) if hasattr(target, "to") else torch.as_tensor(target, device=self.device)
        out = self._eng.step(inp, target)
        self.outputs_buffer.copy_(out.output.reshape(self.outputs_buffer.shape))
        if out.loss is not None:
            self.loss_buffer.fill_(out.loss)
        return out

    __call__ = forward

    def sync_to_net(self):
        """Copy the pipeline's current weights back into the wrapped nn.Sequential."""
        import torch

        model = self._eng.extract_weights()
        mods = list(self.net)
        for mod, spec in zip(mods, model.layers):
            if isinstance(mod, torch.nn.Linear):
                with torch.no_grad():
                    mod.weight.copy_(torch.from_numpy(spec.W))
                    if mod.bias is not None:
                        mod.bias.copy_(torch.from_numpy(spec.b))
        return self.net
