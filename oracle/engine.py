"""engine oracle: the PARTIME lock-step tick on D CPU stages. TEST INFRASTRUCTURE ONLY.

Restates SPEC.md:190-272 with the tick contract pinned in SURVEY.md §8(a).
The contract uses 0-based tick t, 1-based stage h and D stages. Every stage
reads only data produced at tick t-1 (buffer safety):

  (1) in = x_t if h == 1 else inslot_h[(t-1) % 2]   (zeros before first write; Alg. 1 l.1-5)
  (2) forward with the current weights w_h^(t); cache_h[t % 2] holds every
      layer's input (Eq. 6). If h < D, push out -> inslot_{h+1}[t % 2].
  (3) h == D: valid = t >= D-1. If valid, loss = L(out, gamma_{t-D+1}) and
      g = dL/dout; otherwise g = 0 (target queue).
      h < D: g = gslot_h[(t-1) % 2] (Alg. 1 l.9).
  (4) backward with the pre-update weights through cache_h[t % 2] when h == D
      or act_delay == 0. Otherwise (act_delay == 1, the SPEC reading, SPEC.md:196,
      220(d), 256) it uses cache_h[(t-1) % 2]. If h > 1, push
      g_in -> gslot_{h-1}[t % 2] (Eq. 10).
  (5) update iff t >= 2D-h-1 (warm-up policy; Alg. 1 l.12).

Running the stages one after another in any order is equivalent to the SPEC's
D workers between two barriers: within a tick no stage reads
anything written in the same tick. `threads=True` runs them as real workers
with two barriers per tick; that is the CPU baseline's execution mode.
"""

from __future__ import annotations

import threading
from dataclasses import dataclass, field

import numpy as np

from . import netcore as nc


@dataclass
class PipelineOutput:
    """SPEC.md:202-205."""
    step: int
    output: np.ndarray
    loss: float | None
    valid: bool
    source_sample_id: int


@dataclass
class TimelineEvent:
    """(slot, stage, op, sample_id); sample_id < 0 marks a dummy (warm-up) cell."""
    slot: int
    stage: int
    op: str
    sample_id: int


@dataclass
class _Stage:
    h: int
    layers: list
    inslot: list = field(default_factory=lambda: [None, None])
    gslot: list = field(default_factory=lambda: [None, None])
    cache: list = field(default_factory=lambda: [None, None])
    opt: object = None


class Pipeline:
    """CPU PARTIME pipeline over `layers` (oracle tuples), split by `bounds`.

    bounds: D+1 layer indices, bounds[0] = 0, bounds[-1] = len(layers) (StagePlan).
    The layers are used in place: each stage owns its slice.
    """

    def __init__(self, layers, bounds, lr, sample_input, sample_target, loss="mse",
                 optimizer="sgd", act_delay=1, learn=True, threads=False, record_events=False):
        D = len(bounds) - 1
        if D < 1 or bounds[0] != 0 or bounds[-1] != len(layers):
            raise ValueError(f"invalid stage plan {bounds} for {len(layers)} layers")
        if any(bounds[i] >= bounds[i + 1] for i in range(D)):
            raise ValueError(f"stage plan {bounds} has an empty stage")
        self.D, self.loss, self.learn, self.act_delay = D, loss, learn, act_delay
        self.t = 0
        self.events = [] if record_events else None
        self.stages = []
        x = np.zeros_like(np.asarray(sample_input))
        self.dtype = x.dtype
        self.target_queue = {}
        for h in range(1, D + 1):
            sl = layers[bounds[h - 1]:bounds[h]]
            st = _Stage(h=h, layers=sl, opt=nc.make_optimizer(optimizer, lr))
            # shape inference, naming the failing boundary
            try:
                out, inputs = nc.block_forward(sl, x)
            except ValueError as e:
                raise ValueError(f"shape inference failed at stage boundary {h - 1}->{h}: {e}") from None
            zin = np.zeros_like(x)
            st.inslot = [zin.copy(), zin.copy()]
            st.cache = [[np.zeros_like(a) for a in inputs], [np.zeros_like(a) for a in inputs]]
            st.gslot = [np.zeros_like(out), np.zeros_like(out)]
            self.stages.append(st)
            x = out
        if x.shape != np.asarray(sample_target).shape and loss == "mse":
            raise ValueError(f"output shape {x.shape} does not match target shape {np.shape(sample_target)}")
        self.out_shape = x.shape
        self._threads = threads
        self._busy = threading.Lock()
        if threads and D > 1:
            self._start_workers()

    # ---- one stage's share of tick t ---------------------------------------------------------
    def _stage_tick(self, st, t, x_t, res):
        D, h = self.D, st.h
        p, q = t % 2, (t - 1) % 2
        inp = x_t if h == 1 else st.inslot[q]
        out, inputs = nc.block_forward(st.layers, inp)
        # cache_h[t%2] keeps a private copy of the stage input (inslot is rewritten at t+1)
        inputs[0] = np.array(inputs[0], copy=True)
        st.cache[p] = inputs
        if self.events is not None:
            sid = t - h + 1
            res.setdefault("ev", []).append(TimelineEvent(t, h, "F", sid if sid >= 0 else -1))
        if not self.learn:
            if h < D:
                res[("act", h)] = out
            else:
                res["out"] = out
                valid = t >= D - 1
                tgt = self.target_queue.get(t - D + 1)
                if valid and tgt is not None:
                    res["loss"] = nc.loss_eval(self.loss, out, tgt)
            return
        if h == D:
            valid = t >= D - 1
            res["out"] = out
            if valid:
                tgt = self.target_queue[t - D + 1]
                res["loss"] = nc.loss_eval(self.loss, out, tgt)
                g = nc.loss_grad(self.loss, out, tgt)
            else:
                g = np.zeros_like(out)
            cache = st.cache[p]
        else:
            res[("act", h)] = out
            g = st.gslot[q]
            cache = st.cache[q] if self.act_delay == 1 else st.cache[p]
        gin, grads = nc.block_backward(st.layers, cache, g)
        res[("grads", h)] = grads
        if self.events is not None:
            sid = t - 2 * D + h + 1
            res["ev"].append(TimelineEvent(t, h, "B", sid if sid >= 0 else -1))
        if h > 1:
            res[("gin", h)] = gin
        if t >= 2 * D - h - 1:
            nc.apply_updates(st.layers, grads, st.opt)
            if self.events is not None:
                res["ev"].append(TimelineEvent(t, h, "U", t - 2 * D + h + 1))

    def _publish(self, t, res):
        """End-of-step handoff (Alg. 1 l.10 / SPEC.md:261 (2)): write the other parity slots."""
        p = t % 2
        for st in self.stages:
            h = st.h
            if h < self.D:
                self.stages[h].inslot[p] = res[("act", h)]
            if self.learn and h > 1:
                self.stages[h - 2].gslot[p] = res[("gin", h)]

    def step(self, x_t, target_t):
        """pipeline_step."""
        if not self._busy.acquire(blocking=False):
            raise RuntimeError("contract violation: pipeline_step called concurrently (SPEC.md:221)")
        try:
            t = self.t
            x_t = np.asarray(x_t, dtype=self.dtype)
            self.target_queue[t] = np.asarray(target_t) if target_t is not None else None
            res = {}
            if self._threads and self.D > 1:
                self._run_workers(t, x_t, res)
            else:
                for st in self.stages:
                    self._stage_tick(st, t, x_t, res)
            self._publish(t, res)
            self.target_queue.pop(t - self.D + 1, None)
            if self.events is not None:
                self.events.extend(sorted(res.get("ev", []), key=lambda e: (e.stage, "FBU".index(e.op))))
            valid = t >= self.D - 1
            loss = res.get("loss")
            if valid and loss is not None and not np.isfinite(loss):
                raise FloatingPointError(f"non-finite loss at step {t}")
            self.last_grads = {h: res.get(("grads", h)) for h in range(1, self.D + 1)}
            self.t += 1
            return PipelineOutput(step=t, output=res["out"], loss=loss if valid else None,
                                  valid=valid, source_sample_id=t - (self.D - 1))
        finally:
            self._busy.release()

    # ---- D worker threads + two barriers per tick ------------------------------
    def _start_workers(self):
        self._start = threading.Barrier(self.D + 1)
        self._end = threading.Barrier(self.D + 1)
        self._job = None
        self._errors = []
        self._workers = []
        for st in self.stages:
            th = threading.Thread(target=self._worker, args=(st,), daemon=True)
            th.start()
            self._workers.append(th)

    def _worker(self, st):
        while True:
            self._start.wait()
            job = self._job
            if job is None:
                return
            t, x_t, res = job
            local = {}
            try:
                self._stage_tick(st, t, x_t, local)
            except Exception as e:  # surfaced by the driver after the end barrier
                self._errors.append(e)
            with self._lock:
                for k, v in local.items():
                    if k == "ev":
                        res.setdefault("ev", []).extend(v)
                    else:
                        res[k] = v
            self._end.wait()

    _lock = threading.Lock()

    def _run_workers(self, t, x_t, res):
        self._job = (t, x_t, res)
        self._start.wait()
        self._end.wait()
        if self._errors:
            e = self._errors[0]
            self._errors.clear()
            raise e

    def close(self):
        if self._threads and self.D > 1 and self._workers:
            self._job = None
            self._start.wait()
            for th in self._workers:
                th.join()
            self._workers = []

    def extract_weights(self):
        """pipeline_extract_weights: copies of every layer, stage order."""
        out = []
        for st in self.stages:
            for layer in st.layers:
                out.append(tuple([layer[0]] + [np.array(a, copy=True) for a in layer[1:]]))
        return out


def pipeline_run(pipe, xs, ys, n_steps):
    """pipeline_run over in-memory stream arrays; returns the per-step outputs."""
    outs = []
    for t in range(min(n_steps, len(xs))):
        outs.append(pipe.step(xs[t], None if ys is None else ys[t]))
    return outs


def partime_schedule(D, n_steps):
    """schedsim PARTIME rule: at slot t stage h forwards sample t-(h-1)
    and backwards sample t-2D+h+1 (negative ids are warm-up dummies, -1)."""
    ev = []
    for t in range(n_steps):
        for h in range(1, D + 1):
            f = t - h + 1
            b = t - 2 * D + h + 1
            ev.append(TimelineEvent(t, h, "F", f if f >= 0 else -1))
            ev.append(TimelineEvent(t, h, "B", b if b >= 0 else -1))
            if t >= 2 * D - h - 1:
                ev.append(TimelineEvent(t, h, "U", b))
    return ev
