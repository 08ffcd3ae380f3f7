"""B200 PARTIME engine: the reference's `engine` API over the C ABI.

Drop-in for SPEC.md:190-272:
  pipeline_build(model, plan, optimizer, lr, sample_input, sample_target) -> Pipeline
  pipeline_step(pipeline, x_t, target_t) -> PipelineOutput
  pipeline_run(pipeline, stream, n_steps, log_sink) -> RunReport
  pipeline_extract_weights(pipeline) -> Model
Every tick executes in libpartime_b200.so. This module only converts
arguments and copies buffers. The tick semantics are the contract in
SURVEY.md §8(a); `act_delay` selects the SPEC reading (1, the default) or the
paper reading (0).
"""

from __future__ import annotations

import copy as _copy
import ctypes
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .model import Model, StagePlan, canonical_loss, fuse, plan_to_units

try:  # torch is optional for the numpy API; required for device tensors
    import torch
except Exception:  # pragma: no cover
    torch = None


@dataclass
class PipelineOutput:
    """output of step t belongs to sample t-(D-1); valid iff t >= D-1."""
    step: int
    output: object
    loss: float | None
    valid: bool
    source_sample_id: int


@dataclass
class RunReport:
    """per-step records plus wall-clock totals and throughput."""
    steps: list = field(default_factory=list)
    sample_ids: list = field(default_factory=list)
    losses: list = field(default_factory=list)
    valid: list = field(default_factory=list)
    step_wall_seconds: list = field(default_factory=list)
    elapsed: float = 0.0
    outputs: object = None

    @property
    def valid_outputs(self):
        return int(sum(self.valid))

    @property
    def throughput(self):
        return self.valid_outputs / self.elapsed if self.elapsed > 0 else 0.0

    def csv_rows(self):
        yield "step,sample_id,loss,valid,step_wall_seconds"
        for s, i, l, v, w in zip(self.steps, self.sample_ids, self.losses, self.valid, self.step_wall_seconds):
            ls = "" if not v or l is None else f"{l:.9g}"
            yield f"{s},{i},{ls},{int(bool(v))},{w:.9g}"


def _ptr(a):
    if a is None:
        return None
    if torch is not None and isinstance(a, torch.Tensor):
        return ctypes.c_void_p(a.data_ptr())
    return a.ctypes.data_as(ctypes.c_void_p)


def _is_cuda(a):
    return torch is not None and isinstance(a, torch.Tensor) and a.is_cuda


def device_map(devices, D):
    """Stage -> CUDA device ordinal for a `devices` list (one device per stage for
    maximum performance, or fewer, "making multiple stages execute on the same device"). With
    fewer devices than stages, device k takes a contiguous block of stages (k*D//n .. ), so that
    the stages of one device stay contiguous. None -> None (the current device)."""
    if devices is None:
        return None
    devs = list(devices)
    if not devs:
        return None
    if len(devs) > D:
        raise ValueError(f"{len(devs)} devices for {D} stages: at most one device per stage")
    ords = []
    for d in devs:
        if isinstance(d, int):
            ords.append(d)
            continue
        if torch is None:
            raise ValueError(f"device {d!r}: give CUDA device ordinals without torch")
        td = torch.device(d)
        if td.type != "cuda":
            raise ValueError(f"device {d!r} is not a CUDA device (the B200 engine has no CPU path)")
        ords.append(td.index if td.index is not None else torch.cuda.current_device())
    n = len(ords)
    return [ords[h * n // D] for h in range(D)]


def _f32(a):
    if torch is not None and isinstance(a, torch.Tensor):
        return a.detach().to(torch.float32).contiguous()
    return np.ascontiguousarray(np.asarray(a, dtype=np.float32))


class Pipeline:
    """D-stage PARTIME pipeline on B200 (pipeline_build)."""

    def __init__(self, model: Model, plan, optimizer="sgd", lr=1e-3, sample_input=None, sample_target=None,
                 act_delay=1, learn=True, grid=0, local_stages=None, timeout_ms=0, devices=None):
        lib = _lib.load()
        units, owner = fuse(model)
        if isinstance(plan, (list, tuple)):
            plan = StagePlan.from_counts(list(plan))
        sfl = plan_to_units(model, plan, owner)
        dense = [model.layers[u[0]] for u in units]
        dims = [dense[0].in_dim] + [d.out_dim for d in dense]
        for j in range(1, len(dense)):
            if dense[j].in_dim != dims[j]:
                h = next(i for i in range(len(sfl) - 1) if sfl[i] <= j < sfl[i + 1]) + 1
                where = f"stage boundary {h - 1}->{h}" if j == sfl[h - 1] else f"inside stage {h}"
                raise ValueError(f"shape inference failed {where}: layer {units[j][0]} expects "
                                 f"{dense[j].in_dim}, receives {dims[j]} (SPEC.md:212)")
        model.loss = canonical_loss(model.loss)
        if model.loss not in _lib.PT_LOSS:
            raise ValueError(f"unknown loss {model.loss!r}")
        if optimizer not in _lib.PT_OPT:
            raise ValueError(f"unknown optimizer {optimizer!r}")
        si = np.zeros(dims[0], np.float32) if sample_input is None else sample_input
        si_shape = tuple(si.shape)
        if si_shape[-1] != dims[0] or len(si_shape) not in (1, 2):
            raise ValueError(f"shape inference failed at the stage-1 input: sample_input {si_shape} "
                             f"does not end in {dims[0]}")
        self.M = 1 if len(si_shape) == 1 else si_shape[0]
        self._squeeze = len(si_shape) == 1
        # targets: the output vector for mse, one class index per sample for softmax-CE
        self.Fy = 1 if model.loss == "softmax_ce" else dims[-1]
        if sample_target is not None:
            st = tuple(np.shape(sample_target)) if not _is_cuda(sample_target) else tuple(sample_target.shape)
            if int(np.prod(st)) != self.M * self.Fy or (self.Fy > 1 and st[-1] != dims[-1]):
                raise ValueError(f"shape inference failed at the stage-D output: sample_target {st} "
                                 f"vs targets [{self.M}, {self.Fy}]")
        self.model = model
        self.plan = plan
        self.units = units
        self.dims = dims
        self.sfl = sfl
        self.D = len(sfl) - 1
        self.L = len(units)
        self.F = dims[-1]
        self.lr = float(lr)
        self.learn = bool(learn)
        self.act_delay = int(act_delay)
        if local_stages is None:
            local_stages = (0, self.D)
        self.local_first, self.local_count = local_stages
        self.device_of_stage = device_map(devices, self.D)
        dev_i = None if self.device_of_stage is None else (ctypes.c_int32 * self.D)(*self.device_of_stage)
        D_i = (ctypes.c_int32 * len(dims))(*dims)
        A_i = (ctypes.c_int32 * self.L)(*[_lib.PT_ACT[u[1]] for u in units])
        S_i = (ctypes.c_int32 * len(sfl))(*sfl)
        cfg = _lib.PTConfig(
            n_layers=self.L, dims=D_i, act=A_i, loss=_lib.PT_LOSS[model.loss], optimizer=_lib.PT_OPT[optimizer],
            lr=self.lr, n_stages=self.D, stage_first_layer=S_i, batch=self.M, learn=int(self.learn),
            act_delay=self.act_delay, local_stage_first=self.local_first, local_stage_count=self.local_count,
            grid=int(grid), timeout_ms=int(timeout_ms), device_of_stage=dev_i)
        h = ctypes.c_void_p()
        _lib.check(lib.pt_create(ctypes.byref(cfg), ctypes.byref(h)), "pipeline_build")
        self._h = h
        # devices of this process's stages (several: one handle drives one part per device)
        local = range(self.local_first + 1, self.local_first + self.local_count + 1)
        self.stage_devices = {s: int(lib.pt_stage_device(h, s)) for s in local}
        # one handle driving several devices (PT_VIRTUAL_DEVICES may map them onto one GPU, so
        # this follows the requested map; stage_devices holds the physical ordinals)
        self.multi_device = self.device_of_stage is not None and len(
            {self.device_of_stage[s - 1] for s in local}) > 1
        self._lib = lib
        self._t = 0
        self._user_stream = False
        lo, hi = sfl[self.local_first], sfl[self.local_first + self.local_count]
        for j in range(lo, hi):
            self.set_layer(j, dense[j].W, dense[j].b)

    # ---- parameters ----------------------------------------------------------------------
    def _local_units(self):
        return range(self.sfl[self.local_first], self.sfl[self.local_first + self.local_count])

    def set_layer(self, j, W, b):
        """Upload fused layer j's parameters (W [out, in], b [out])."""
        if W is None or b is None:
            raise ValueError(f"layer {self.units[j][0]} has no weights (run init_weights first)")
        W, b = _f32(W), _f32(b)
        where = _lib.PT_DEVICE if _is_cuda(W) else _lib.PT_HOST
        _lib.check(self._lib.pt_set_params(self._h, j, _ptr(W), _ptr(b), where), "set_params")

    def get_layer(self, j):
        n_out, n_in = self.dims[j + 1], self.dims[j]
        W = np.empty((n_out, n_in), np.float32)
        b = np.empty(n_out, np.float32)
        _lib.check(self._lib.pt_get_params(self._h, j, _ptr(W), _ptr(b), _lib.PT_HOST), "extract_weights")
        return W, b

    def extract_weights(self) -> Model:
        """pipeline_extract_weights: current weights, stamped with
        the number of updates their stage has applied (the w_h^(t) version of Eq. 7)."""
        m = _copy.copy(self.model)
        m.layers = [_copy.copy(l) for l in self.model.layers]
        local = set(self._local_units())
        for j, (idx, _) in enumerate(self.units):
            if j not in local:
                continue
            W, b = self.get_layer(j)
            h = next(s for s in range(self.D) if self.sfl[s] <= j < self.sfl[s + 1]) + 1
            m.layers[idx].W, m.layers[idx].b = W, b
            m.layers[idx].version = max(0, self._t - (2 * self.D - h - 1)) if self.learn and self.lr else 0
        return m

    # ---- ticks ---------------------------------------------------------------------------
    @property
    def t(self):
        return self._t

    def timeline(self, n_samples=None):
        """TimelineEvents (schedsim.TimelineEvent) of the ticks run so far on this process's
        stages, for the engine/simulator agreement check. Tick t of stage h
        forwards the activation stage h-1 produced at tick t-1 (the kernel polls inslot for
        tag t-1; stage 1 reads x_t) and backwards the gradient stage h+1 produced at tick t-1
        (gslot tag t-1; stage D uses its own tick's loss gradient), so by induction F is
        sample t-(h-1) and B is sample t-2D+h+1; the update follows B on every learning tick.
        Events whose sample is negative (warm-up) or >= n_samples are omitted."""
        from .schedsim import TimelineEvent
        ev = []
        for t in range(self._t):
            for h in range(self.local_first + 1, self.local_first + self.local_count + 1):
                kf, kb = t - (h - 1), t - 2 * self.D + h + 1
                if kf >= 0 and (n_samples is None or kf < n_samples):
                    ev.append(TimelineEvent(t, h, "F", kf))
                if self.learn and kb >= 0 and (n_samples is None or kb < n_samples):
                    ev.append(TimelineEvent(t, h, "B", kb))
                    ev.append(TimelineEvent(t, h, "U", kb))
        return ev

    def step(self, x_t, target_t=None) -> PipelineOutput:
        """pipeline_step: one synchronous tick."""
        if type(x_t) is np.ndarray and (target_t is None or type(target_t) is np.ndarray):
            return self._step_host(x_t, target_t)
        M, F = self.M, self.F
        dev = _is_cuda(x_t) or _is_cuda(target_t)
        x = None if x_t is None else _f32(x_t)
        y = None if target_t is None else _f32(target_t)
        if x is not None and int(np.prod(tuple(x.shape))) != M * self.dims[0]:
            raise ValueError(f"x_t has shape {tuple(x.shape)}, expected [{M}, {self.dims[0]}]")
        if y is not None and int(np.prod(tuple(y.shape))) != M * self.Fy:
            raise ValueError(f"target_t has shape {tuple(y.shape)}, expected [{M}, {self.Fy}]")
        if y is not None and not dev:
            self._check_targets(y, f"step {self._t}")
        if dev:
            x, y = self._place(x, y)
            out = torch.empty((M, F), dtype=torch.float32, device=self._out_device(x, y))
            loss = torch.empty(1, dtype=torch.float32, device=out.device)
            valid = torch.empty(1, dtype=torch.int32, device=out.device)
            where = _lib.PT_DEVICE
        else:
            out = np.empty((M, F), np.float32)
            loss = np.empty(1, np.float32)
            valid = np.empty(1, np.int32)
            where = _lib.PT_HOST
        order = dev and not self._user_stream
        if order:
            self._order_after_torch(out.device)
        rc = self._lib.pt_step(self._h, _ptr(x), _ptr(y), _ptr(out), _ptr(loss), _ptr(valid), where)
        if order:
            self._order_torch_after(out.device)
        t = self._t
        self._t += 1
        _lib.check(rc, f"pipeline_step at step {t}")
        has_last = self.local_first + self.local_count == self.D
        v = bool(int(valid[0])) if has_last else t >= self.D - 1
        lval = float(loss[0]) if (has_last and v and y is not None) else None
        o = out[0] if self._squeeze else out
        return PipelineOutput(step=t, output=o, loss=lval, valid=v, source_sample_id=t - (self.D - 1))

    def _step_host(self, x_t, target_t):
        """The per-sample host path with as little Python as possible: the library serves
        consecutive steps from one resident launch, so the call overhead is the step's cost."""
        M, F = self.M, self.F
        x = x_t if (x_t.dtype == np.float32 and x_t.flags.c_contiguous) else _f32(x_t)
        if x.size != M * self.dims[0]:
            raise ValueError(f"x_t has shape {tuple(x.shape)}, expected [{M}, {self.dims[0]}]")
        y = None
        if target_t is not None:
            y = target_t if (target_t.dtype == np.float32 and target_t.flags.c_contiguous) else _f32(target_t)
            if y.size != M * self.Fy:
                raise ValueError(f"target_t has shape {tuple(y.shape)}, expected [{M}, {self.Fy}]")
            if self.Fy == 1:
                self._check_targets(y, f"step {self._t}")
        out = np.empty((M, F), np.float32)
        sc = getattr(self, "_scalars", None)
        if sc is None:
            sc = self._scalars = (np.empty(1, np.float32), np.empty(1, np.int32))
        loss, valid = sc
        rc = self._lib.pt_step(self._h, x.ctypes.data, None if y is None else y.ctypes.data, out.ctypes.data,
                               loss.ctypes.data, valid.ctypes.data, _lib.PT_HOST)
        t = self._t
        self._t += 1
        if rc:
            _lib.check(rc, f"pipeline_step at step {t}")
        has_last = self.local_first + self.local_count == self.D
        v = bool(valid[0]) if has_last else t >= self.D - 1
        lval = float(loss[0]) if (has_last and v and y is not None) else None
        return PipelineOutput(step=t, output=out[0] if self._squeeze else out, loss=lval, valid=v,
                              source_sample_id=t - (self.D - 1))

    def run(self, xs, ys=None, n=None):
        """n ticks with no per-tick host round trip (pt_run). xs [n, M, d0], ys [n, M, F]
        (mse) or [n, M] class indices (softmax_ce).
        numpy inputs take the host path; CUDA tensors run asynchronously on the device.
        Returns (outs [n, M, F], losses [n], valid [n])."""
        n = int(n if n is not None else (xs.shape[0] if xs is not None else ys.shape[0]))
        M, F = self.M, self.F
        dev = _is_cuda(xs) or _is_cuda(ys) or (xs is None and ys is None and torch is not None)
        xs = None if xs is None else _f32(xs)
        ys = None if ys is None else _f32(ys)
        if ys is not None and not dev:
            self._check_targets(ys, f"steps [{self._t}, {self._t + n})")
        if dev:
            xs, ys = self._place(xs, ys)
            d = self._out_device(xs, ys)
            outs = torch.empty((n, M, F), dtype=torch.float32, device=d)
            losses = torch.empty(n, dtype=torch.float32, device=d)
            valid = torch.empty(n, dtype=torch.uint8, device=d)
            where = _lib.PT_DEVICE
        else:
            outs = np.empty((n, M, F), np.float32)
            losses = np.empty(n, np.float32)
            valid = np.empty(n, np.uint8)
            where = _lib.PT_HOST
        has_last = self.local_first + self.local_count == self.D
        t0 = self._t
        if not has_last:
            # this process does not own stage D: no outputs or losses here, but validity is
            # known from the tick alone. Filled before the launch: a torch
            # kernel launched while the pipeline runs may need a lazy module load, which waits
            # for the running kernels, while they wait for a neighbour that has not launched yet
            ticks = np.arange(t0, t0 + n)
            if dev:
                valid.copy_(torch.from_numpy((ticks >= self.D - 1).astype(np.uint8)))
                losses.fill_(float("nan"))
                outs.fill_(float("nan"))
            else:
                valid[:] = ticks >= self.D - 1
                losses[:] = np.nan
                outs[:] = np.nan
        order = dev and not self._user_stream
        if order:
            self._order_after_torch(outs.device)
        rc = self._lib.pt_run(self._h, _ptr(xs), _ptr(ys), n, _ptr(outs) if has_last else None,
                              _ptr(losses) if has_last else None, _ptr(valid) if has_last else None, where)
        if order:
            self._order_torch_after(outs.device)
        self._t += n
        _lib.check(rc, f"pipeline_run at steps [{t0}, {t0 + n})")
        return outs, losses, valid

    def _check_targets(self, y, where):
        """softmax-CE targets are class indices in [0, F). Host arrays are
        checked here; device targets are checked by the kernel (PT_EINVAL at sync)."""
        if self.model.loss != "softmax_ce":
            return
        y = np.asarray(y)
        bad = ~((y >= 0) & (y < self.F) & (y == np.floor(y)))
        if bad.any():
            raise ValueError(f"target out of class range for cross-entropy at {where}: "
                             f"{y.reshape(-1)[np.argmax(bad.reshape(-1))]!r} not in [0, {self.F})")

    def sync(self):
        _lib.check(self._lib.pt_sync(self._h), "sync")

    # ---- stream ordering with torch (device buffers) ---------------------------------------
    def _place(self, x, y):
        """Device inputs of a multi-device pipeline: x on stage 1's device, targets on stage D's."""
        if not self.multi_device:
            return x, y
        if x is not None and 1 in self.stage_devices:
            x = x.to(torch.device("cuda", self.stage_devices[1]))
        if y is not None and self.D in self.stage_devices:
            y = y.to(torch.device("cuda", self.stage_devices[self.D]))
        return x, y

    def _out_device(self, x, y):
        if self.D in self.stage_devices:
            return torch.device("cuda", self.stage_devices[self.D])
        if x is not None:
            return x.device
        return y.device if y is not None else torch.device("cuda", torch.cuda.current_device())

    def _stream(self, device):
        raw = ctypes.c_void_p()
        _lib.check(self._lib.pt_get_stream(self._h, ctypes.byref(raw)), "get_stream")
        return torch.cuda.ExternalStream(raw.value or 0, device=device)

    def _order_after_torch(self, device):
        """Device inputs were written on torch's current stream (e.g. an async H2D copy):
        the handle's stream waits for it before the kernel reads them. A multi-device handle
        runs one private stream per device: torch's streams on those devices are drained."""
        if self.multi_device:
            for d in sorted(set(self.stage_devices.values())):
                torch.cuda.current_stream(torch.device("cuda", d)).synchronize()
            return
        self._stream(device).wait_stream(torch.cuda.current_stream(device))

    def _order_torch_after(self, device):
        """Outputs are written on the handle's stream: torch's current stream waits for them."""
        torch.cuda.current_stream(device).wait_stream(self._stream(device))

    def set_stream(self, stream):
        """Run on an external CUDA stream (torch.cuda.Stream or raw handle). The caller then
        owns the ordering of device buffers against its other streams (e.g. two co-resident
        stage handles on two streams must stay concurrent); with the private stream (None)
        the engine orders itself after torch's current stream and torch's after the run."""
        raw = getattr(stream, "cuda_stream", stream)
        _lib.check(self._lib.pt_set_stream(self._h, ctypes.c_void_p(raw) if raw else None), "set_stream")
        self._user_stream = bool(raw)

    @property
    def kernel_path(self):
        """'panel' (batch-1 panel kernel, SGD or Adam), 'tile' (tcgen05 tensor-core tile kernel, micro-batch 16/32/64)
        or 'tick' (row-owned SIMT tick kernel, every other case)."""
        r = self._lib.pt_kernel_path(self._h)
        if r < 0:
            _lib.check(r, "kernel_path")
        return {0: "tick", 1: "tile", 2: "panel"}[r]

    def last_kernel_ms(self):
        ms = ctypes.c_float()
        _lib.check(self._lib.pt_last_kernel_ms(self._h, ctypes.byref(ms)), "last_kernel_ms")
        return float(ms.value)

    def set_trace(self, cta=0, cap=1 << 16):
        """Diagnostics: record device timestamps of one CTA's step phases (pt_set_trace)."""
        _lib.check(self._lib.pt_set_trace(self._h, int(cta), int(cap)), "set_trace")
        self._trace_cap = int(cap)

    def get_trace(self):
        """(consumer, producer) lists of (code, ns) from the last run."""
        buf = np.zeros(self._trace_cap, np.uint64)
        _lib.check(self._lib.pt_get_trace(self._h, _ptr(buf), self._trace_cap), "get_trace")
        half, q = self._trace_cap // 2, self._trace_cap - self._trace_cap // 4
        dec = lambda a: [(int(v >> np.uint64(56)), int(v & np.uint64(0x00FFFFFFFFFFFFFF))) for v in a if v]
        return dec(buf[:half]), dec(buf[half:q]), dec(buf[q:])

    # ---- multi-process (one process per GPU) ----------------------------------------------
    def ipc_export(self, stage):
        buf = ctypes.create_string_buffer(256)
        n = ctypes.c_size_t()
        _lib.check(self._lib.pt_ipc_export(self._h, stage, buf, 256, ctypes.byref(n)), "ipc_export")
        return buf.raw[:n.value]

    def ipc_import(self, blob: bytes):
        b = ctypes.create_string_buffer(blob, len(blob))
        _lib.check(self._lib.pt_ipc_import(self._h, b, len(blob)), "ipc_import")

    def close(self):
        if getattr(self, "_h", None):
            self._lib.pt_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---- SPEC function-style API -----------------------------------------------------------------

def pipeline_build(model, plan, optimizer="sgd", lr=1e-3, sample_input=None, sample_target=None, **kw):
    """SPEC.md:208-216."""
    return Pipeline(model, plan, optimizer, lr, sample_input, sample_target, **kw)


def pipeline_step(pipeline, x_t, target_t=None):
    """SPEC.md:217-225."""
    return pipeline.step(x_t, target_t)


def pipeline_run(pipeline, stream, n_steps, log_sink=None, chunk=256):
    """drive n_steps ticks from `stream`, in chunks of device-resident ticks.

    Streams with .block(t0, n) hand over arrays directly. Any other iterator of
    (x, gamma[, id]) is batched per chunk. Exhaustion stops cleanly with a partial report.
    """
    rep = RunReport()
    done = 0
    t_start = time.perf_counter()
    outs_all = []
    while done < n_steps:
        n = min(chunk, n_steps - done)
        if hasattr(stream, "block"):
            t_s = getattr(stream, "t", done)
            if hasattr(stream, "__len__"):
                # finite stream (replay over a DatasetFile): stop cleanly at its end with a
                # partial report
                n = min(n, len(stream) - t_s)
                if n <= 0:
                    break
            xs, ys = stream.block(t_s, n)
            if hasattr(stream, "t"):
                stream.t += n
        else:
            xb, yb = [], []
            for _ in range(n):
                try:
                    item = next(stream)
                except StopIteration:
                    break
                xb.append(np.asarray(item[0], np.float32).reshape(pipeline.M, -1))
                yb.append(np.asarray(item[1], np.float32).reshape(pipeline.M, -1))
            if not xb:
                break
            xs, ys = np.stack(xb), np.stack(yb)
            n = len(xb)
        c0 = time.perf_counter()
        t0 = pipeline.t
        outs, losses, valid = pipeline.run(np.asarray(xs, np.float32), np.asarray(ys, np.float32), n)
        dt = (time.perf_counter() - c0) / n
        outs_all.append(outs)
        for i in range(n):
            t = t0 + i
            v = bool(valid[i])
            rep.steps.append(t)
            rep.sample_ids.append(t - (pipeline.D - 1))
            rep.losses.append(float(losses[i]) if (v and np.isfinite(losses[i])) else None)
            rep.valid.append(v)
            rep.step_wall_seconds.append(dt)
        done += n
        if n < chunk and (not hasattr(stream, "block") or hasattr(stream, "__len__")):
            break
    rep.elapsed = time.perf_counter() - t_start
    rep.outputs = np.concatenate(outs_all) if outs_all else None
    if log_sink is not None:
        for row in rep.csv_rows():
            log_sink(row) if callable(log_sink) else log_sink.write(row + "\n")
    return rep


def pipeline_extract_weights(pipeline):
    """SPEC.md:235-243."""
    return pipeline.extract_weights()
