"""Schedule simulator (reference `schedsim` module).

Deterministic, unit-cost slot model of four pipeline policies:
- partime: every stage runs one PARTIME step per slot (forward, backward and
  update of its layer slice, PAPER Fig. 3). At slot t stage h (1-based)
  forwards sample t-(h-1) and backwards sample t-2D+h+1 when those exist
  (SPEC.md:293, 299). This is the rule the B200 tick kernel executes: stage h
  reads the activation stage h-1 wrote at tick t-1 (pt_kernels.cuh, inslot
  tag t-1) and the gradient stage h+1 wrote at tick t-1.
- gpipe: m micro-batches forward, then backward, then a synchronised update
  (pipeline flush, PAPER §2). F and B each take one slot.
- pipedream: 1F1B with weight stashing; stage h admits at most D-h+1
  samples in flight (PAPER §2, "D - s + 1").
- pipedream2bw: the 1F1B schedule with a weight update every m backward
  passes and a one-version delay (two stored versions, PAPER §2).

Throughput is counted in samples per slot in the steady state, where a slot
is one stage step: one PARTIME step, or one F or one B of the other policies.
The sequential baseline takes D slots per sample.

Staleness[h] is the number of weight updates stage h applies between F_h(k)
and B_h(k) (the max over steady-state samples): 2(D-h) for partime (one
update per slot), 0 at stage D of a 1F1B schedule.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from fractions import Fraction

POLICIES = ("gpipe", "pipedream", "pipedream2bw", "partime")


@dataclass
class SchedulePolicy:
    """SPEC.md:279-282."""
    kind: str
    D: int
    n: int = 8            # samples (steps) to simulate
    m: int = 4            # micro-batches per mini-batch (gpipe, 2bw)
    update_slots: int = 0  # slots a gpipe update takes (zero by default)

    def validate(self):
        if self.kind not in POLICIES:
            raise ValueError(f"unknown policy {self.kind!r} (one of {', '.join(POLICIES)})")
        if self.D < 1:
            raise ValueError("D must be >= 1")
        if self.n < 0:
            raise ValueError("n must be >= 0")
        if self.kind in ("gpipe", "pipedream", "pipedream2bw") and self.m < 1:
            raise ValueError("m must be >= 1")
        if self.kind == "pipedream2bw" and self.m < self.D:
            raise ValueError(f"pipedream2bw requires m >= D (m={self.m}, D={self.D})")


@dataclass(frozen=True)
class TimelineEvent:
    """SPEC.md:283-286. stage is 1-based; sample is the sample / micro-batch id (-1 for U
    of gpipe, which updates on the whole mini-batch)."""
    slot: int
    stage: int
    op: str
    sample: int = -1


@dataclass
class ScheduleReport:
    """SPEC.md:287-290."""
    throughput: Fraction
    idle_fraction: list
    staleness: list
    weight_versions: list
    activation_stash: list
    slots: int = 0
    extra: dict = field(default_factory=dict)

    def as_dict(self):
        return {"throughput": float(self.throughput), "throughput_exact": str(self.throughput),
                "idle_fraction": [float(f) for f in self.idle_fraction], "staleness": self.staleness,
                "weight_versions": self.weight_versions, "activation_stash": self.activation_stash,
                "slots": self.slots}


# ---------------------------------------------------------------------------- schedules

def _partime(D, n):
    ev = []
    for t in range(n + 2 * D - 2):
        for h in range(1, D + 1):
            kf, kb = t - (h - 1), t - 2 * D + h + 1
            if 0 <= kf < n:
                ev.append(TimelineEvent(t, h, "F", kf))
            if 0 <= kb < n:
                ev.append(TimelineEvent(t, h, "B", kb))
                ev.append(TimelineEvent(t, h, "U", kb))
    return ev


def _gpipe(D, n, m, u):
    ev, t0 = [], 0
    for b0 in range(0, n, m):
        mb = list(range(b0, min(n, b0 + m)))
        q = len(mb)
        for j, k in enumerate(mb):
            for h in range(1, D + 1):
                ev.append(TimelineEvent(t0 + j + h - 1, h, "F", k))
        tb = t0 + q + D - 1
        for j, k in enumerate(reversed(mb)):
            for h in range(D, 0, -1):
                ev.append(TimelineEvent(tb + j + (D - h), h, "B", k))
        tu = tb + q + D - 1
        for h in range(1, D + 1):  # the flush: every stage updates together
            for s in range(max(u, 1)):
                ev.append(TimelineEvent(tu + s, h, "U", -1))
        t0 = tu + u
    return ev


def _one_f_one_b(D, n):
    """Event-driven 1F1B: a ready B first, else a ready F while fewer than D-h+1 samples are
    in flight at stage h; an op's result is visible to the neighbour from the next slot."""
    f_done = [dict() for _ in range(D + 2)]   # stage -> {sample: slot}
    b_done = [dict() for _ in range(D + 2)]
    next_f = [0] * (D + 2)
    next_b = [0] * (D + 2)
    ev, t = [], 0
    while next_b[1] < n:
        acts = []
        for h in range(1, D + 1):
            kb, kf = next_b[h], next_f[h]
            b_ready = kb < next_f[h] and (
                (h == D and f_done[h].get(kb, t) < t) or (h < D and b_done[h + 1].get(kb, t) < t))
            f_ready = kf < n and (h == 1 or f_done[h - 1].get(kf, t) < t)
            if b_ready:
                acts.append((h, "B", kb))
            elif f_ready and next_f[h] - next_b[h] < D - h + 1:
                acts.append((h, "F", kf))
        for h, op, k in acts:
            ev.append(TimelineEvent(t, h, op, k))
            if op == "F":
                f_done[h][k] = t
                next_f[h] += 1
            else:
                b_done[h][k] = t
                next_b[h] += 1
        t += 1
        if t > 4 * (n + D) + 16:
            raise RuntimeError("1F1B simulation did not converge")
    return ev


def _with_updates(ev, D, every):
    """Add a zero-slot U after every `every`-th backward of each stage (pipedream: 1)."""
    out, cnt = [], [0] * (D + 1)
    for e in ev:
        out.append(e)
        if e.op == "B":
            cnt[e.stage] += 1
            if cnt[e.stage] % every == 0:
                out.append(TimelineEvent(e.slot, e.stage, "U", e.sample))
    return out


def _events(p: SchedulePolicy):
    if p.kind == "partime":
        return _partime(p.D, p.n)
    if p.kind == "gpipe":
        return _gpipe(p.D, p.n, p.m, p.update_slots)
    base = _one_f_one_b(p.D, p.n)
    return _with_updates(base, p.D, 1 if p.kind == "pipedream" else p.m)


# ---------------------------------------------------------------------------- metrics

def _check_causality(ev, D, n):
    f = {(e.stage, e.sample): e.slot for e in ev if e.op == "F"}
    b = {(e.stage, e.sample): e.slot for e in ev if e.op == "B"}
    if n and (len(f) != D * n or len(b) != D * n):
        raise AssertionError("every sample must be forwarded and backwarded once per stage")
    for k in range(n):
        for h in range(1, D):
            assert f[(h, k)] < f[(h + 1, k)], ("F order", h, k)
            assert b[(h + 1, k)] < b[(h, k)], ("B order", h, k)
        assert f[(D, k)] <= b[(D, k)]
    return f, b


def _report(p: SchedulePolicy, ev):
    D, n = p.D, p.n
    f, b = _check_causality(ev, D, n)
    slots = 1 + max((e.slot for e in ev), default=-1)
    # update counts per stage by slot: an update at slot s is seen by F/B in later slots;
    # for partime the update of slot s follows that slot's F and B
    ups = {h: sorted(e.slot for e in ev if e.op == "U" and e.stage == h) for h in range(1, D + 1)}

    def n_updates(h, t0, t1):  # updates applied after the op at t0 and before the op at t1
        if p.kind == "partime":  # a PARTIME slot's update follows its F and B
            return sum(1 for s in ups[h] if t0 <= s < t1)
        return sum(1 for s in ups[h] if t0 < s < t1)  # U rides on a B slot (or its own slots)

    staleness, versions, stash = [], [], []
    for h in range(1, D + 1):
        st = [n_updates(h, f[(h, k)], b[(h, k)]) for k in range(n)]
        staleness.append(max(st[len(st) // 2:], default=0))
        if p.kind == "partime":
            versions.append(1)  # no stashing: the backward uses the current weights (Eq. 9-10)
            stash.append(1)
            continue
        # stored versions: the versions in-flight samples were forwarded with, plus the current one
        vmax, smax = 1, 0
        for t in range(slots):
            inflight = [k for k in range(n) if f[(h, k)] <= t < b[(h, k)]]
            vers = {_version_at(ups[h], f[(h, k)]) for k in inflight} | {_version_at(ups[h], t + 1)}
            vmax = max(vmax, len(vers))
            smax = max(smax, len(inflight))
        if p.kind == "pipedream2bw":  # W(t+1) = W(t) - lr grad f(W(t-1)): both are kept
            vmax = max(vmax, 2)
        versions.append(vmax if p.kind != "gpipe" else 1)
        stash.append(smax)
    thr, idle = _steady_state(p)
    return ScheduleReport(thr, idle, staleness, versions, stash, slots)


def _version_at(up_slots, t):
    """Number of updates at the stage that completed before slot t."""
    return sum(1 for s in up_slots if s < t)


def _steady_state(p: SchedulePolicy):
    """Exact steady-state throughput and per-stage idle fraction, from a long run."""
    D = p.D
    period = p.m if p.kind == "gpipe" else 1
    n = 8 * (D + p.m) * max(1, period)
    n -= n % period
    q = SchedulePolicy(p.kind, D, n, p.m, p.update_slots)
    ev = _events(q)
    done = {}
    for e in ev:
        if e.op == "B" and e.stage == 1:
            done[e.sample] = e.slot
    # a window of whole periods in the middle of the run: no fill, no drain
    k0 = (n // 4) - (n // 4) % period - 1
    k1 = (n // 2) - (n // 2) % period - 1
    t0, t1 = done[k0], done[k1]
    if p.kind == "gpipe":  # a period ends with the flush update
        t0 += D - 1 + p.update_slots
        t1 += D - 1 + p.update_slots
    thr = Fraction(k1 - k0, t1 - t0)
    busy = {h: set() for h in range(1, D + 1)}
    for e in ev:
        if t0 < e.slot <= t1 and (e.op in ("F", "B") or (e.op == "U" and p.kind == "gpipe" and p.update_slots)):
            busy[e.stage].add(e.slot)
    idle = [Fraction(t1 - t0 - len(busy[h]), t1 - t0) for h in range(1, D + 1)]
    return thr, idle


def simulate(policy: SchedulePolicy):
    """(events, report)."""
    policy.validate()
    ev = _events(policy)
    return ev, _report(policy, ev)


def render_timeline(events, D, width=0):
    """one row per stage, one column per slot. A PARTIME cell is the
    slot's forward then backward (+ U), '-' where the stage has no real sample."""
    slots = 1 + max((e.slot for e in events), default=-1)
    if width:
        slots = min(slots, width)
    cells = [[[] for _ in range(slots)] for _ in range(D)]
    for e in events:
        if e.slot < slots:
            cells[e.stage - 1][e.slot].append(e)
    partime = any(e.op == "F" and any(x.op == "B" and x.slot == e.slot and x.stage == e.stage for x in events)
                  for e in events)

    def cell(es):
        if not es:
            return "--" if partime else "-"
        out = ""
        ops = {e.op: e for e in es}
        if partime:
            out += f"F{ops['F'].sample}" if "F" in ops else "-"
            out += f"B{ops['B'].sample}" if "B" in ops else "-"
            return out + ("U" if "U" in ops else "")
        flush = "U" in ops and ops["U"].sample < 0  # gpipe's update precedes the next mini-batch
        for op in ("F", "B"):
            if op in ops:
                out += f"{op}{ops[op].sample}"
        return ("U" + out) if flush else out + ("U" if "U" in ops else "")

    grid = [[cell(cells[h][t]) for t in range(slots)] for h in range(D)]
    w = max((len(c) for row in grid for c in row), default=1)
    return "\n".join(f"{h + 1:>2} | " + " ".join(c.ljust(w) for c in row) for h, row in enumerate(grid))


def compare_policies(policies, n=None):
    """one row per policy."""
    rows = []
    for p in policies:
        if n is not None:
            p = SchedulePolicy(p.kind, p.D, n, p.m, p.update_slots)
        _, r = simulate(p)
        rows.append({"policy": p.kind, "D": p.D, "m": p.m, "throughput": float(r.throughput),
                     "idle": float(max(r.idle_fraction)), "staleness_max": max(r.staleness),
                     "weight_versions_max": max(r.weight_versions), "activation_stash_max": max(r.activation_stash)})
    return rows
