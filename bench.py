"""Benchmark: stream samples/s of the PARTIME per-tick pipeline on B200.

The workload is BASELINE.json configs[1] (C2): a 32-layer, 2048-wide ReLU MLP,
online learning, batch 1, on the synthetic smooth stream.
With N GPUs it runs D = N stages, one per GPU and one process per GPU
(torchrun), and activations and gradients move by NVLink peer stores.
One bench step is one pt_run call of --ticks ticks, i.e. that many stream
samples, with every input already resident in HBM.

Output is one JSON line on rank 0, following the driver contract. It includes
`roofline` (dominant kernel = the tick kernel vs measured HBM bandwidth),
`cpu_baseline` (the numpy oracle on this host's cores), `e2e` (the public API
with pinned host buffers and host<->device copies in the timed region) and
`clocks`. `--impl reference` times the reference CPU path (the oracle port)
on the same config instead.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WIDTH, LAYERS, BATCH = 2048, 32, 1
METRIC = "stream samples/sec (online learning)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--ticks", type=int, default=64, help="stream ticks (samples) per bench step")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--width", type=int, default=WIDTH)
    ap.add_argument("--layers", type=int, default=LAYERS)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="budget of the cpu_baseline sample")
    ap.add_argument("--no-extra", action="store_true", help="skip the other BASELINE configs (N=1 only)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("PT_BENCH_ONE_DEVICE"):  # test hook: all ranks share GPU 0 (time-sliced)
        local = 0
    return rank, world, local


def plan_counts(L, D):
    """Equal split of L dense+ReLU units into D stages, in SPEC layer counts (the last
    unit has no activation)."""
    per = [L // D + (1 if i < L % D else 0) for i in range(D)]
    counts, u = [], 0
    for c in per:
        counts.append(sum(2 if (u + j) < L - 1 else 1 for j in range(c)))
        u += c
    return counts


def algorithmic_bytes_per_tick(widths, learn=True, optimizer="sgd"):
    """learn Σ(12·n_in·n_out + 4·n_out), infer Σ 4·n_in·n_out (fp32). Adam reads
    and writes its two moments too: Σ(28·n_in·n_out + 20·n_out) (optimizer row)."""
    w_b, b_b = (28, 20) if optimizer == "adam" else (12, 4)
    tot = 0
    for i in range(len(widths) - 1):
        tot += (w_b if learn else 4) * widths[i] * widths[i + 1] + (b_b * widths[i + 1] if learn else 0)
    return tot


class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.rows, self.proc = index, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def cpu_reference(widths, D, ticks_budget_s, steps=None, warmup=0, ticks_per_step=None):
    """Time the oracle (numpy f32 + OpenBLAS) on the same config: D = 1 gives BLAS every host
    core; D > 1 runs BASELINE.md §3's threaded pipeline (one worker thread per stage, two
    barriers per tick) with floor(cores / D) BLAS threads per worker
    (`tools/cpu_scaling.py` measures D = 1, 2, 4, 8).

    Returns (samples/s, cores, sample description, per-step seconds).
    """
    from oracle import engine as oeng
    from paper_2210_09147_b200 import model as mdl, streams
    cores = len(os.sched_getaffinity(0))
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(max(1, cores // D))
    except Exception:
        pass
    m = mdl.mlp(widths, seed=0, dtype=np.float32)
    layers = [("dense", l.W, l.b) if l.kind == "dense" else (l.kind,) for l in m.layers]
    counts = plan_counts(len(widths) - 1, D)
    bounds = [0]
    for c in counts:
        bounds.append(bounds[-1] + c)
    st = streams.SmoothStream(widths[0], widths[-1], seed=1)
    p = oeng.Pipeline(layers, bounds, 1e-3, np.zeros((1, widths[0]), np.float32), np.zeros((1, widths[-1]), np.float32),
                      threads=D > 1)
    xs, ys = st.block(0, 64)
    xs, ys = xs.astype(np.float32), ys.astype(np.float32)
    t = 0
    for _ in range(max(1, warmup)):  # warm-up tick(s)
        p.step(xs[t % 64], ys[t % 64])
        t += 1
    times = []
    if steps is None:  # bounded sample: as many ticks as fit in the budget
        t0 = time.perf_counter()
        n = 0
        while time.perf_counter() - t0 < ticks_budget_s:
            p.step(xs[t % 64], ys[t % 64])
            t += 1
            n += 1
        el = time.perf_counter() - t0
        p.close()
        return n / el, cores, f"{n} ticks of C2 (D={D}) in {el:.1f}s, numpy f32 + OpenBLAS ({max(1, cores // D)} threads x {D})", [el]
    for _ in range(steps):
        t0 = time.perf_counter()
        for _ in range(ticks_per_step):
            p.step(xs[t % 64], ys[t % 64])
            t += 1
        times.append(time.perf_counter() - t0)
    p.close()
    n = steps * ticks_per_step
    return n / sum(times), cores, f"{ticks_per_step} ticks/step of C2 (D={D}), numpy f32 + OpenBLAS ({max(1, cores // D)} threads x {D})", times


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    widths = [args.width] * (args.layers + 1)
    D = world if world > 1 else args.gpus if args.gpus > 1 else 1
    # each step is a bounded sample: a few ticks so K+W steps finish in minutes
    tps = max(1, int(os.environ.get("PT_REF_TICKS", "2")))
    value, cores, sample, times = cpu_reference(widths, D, 0, steps=args.steps, warmup=args.warmup,
                                                ticks_per_step=tps)
    ms = 1e3 * statistics.mean(times)
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "fp32", "data": "synthetic smooth-d stream",
        "config": {"workload": f"C2: {args.layers}-layer {args.width}-wide ReLU MLP, online learning, batch 1",
                   "stages": D, "ticks_per_step": tps},
        "cpu_baseline": {"value": value, "unit": "samples/s", "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def balanced_counts(widths, D, learn):
    from paper_2210_09147_b200 import partition
    L = len(widths) - 1
    costs, _ = partition.mlp_costs(widths, learn)
    units, _ = partition.balance(costs, D)
    out, u = [], 0
    for c in units:
        out.append(sum(2 if (u + j) < L - 1 else 1 for j in range(c)))
        u += c
    return out


def extra_configs(peak):
    """Device time per tick of the other BASELINE.json configs on this one GPU (all stages
    here): C3 inference wave, C4 micro-batch 16 and 32 (tcgen05 tile kernel), C5 uneven widths.
    Reported beside the headline line; not part of `value`."""
    import torch
    from paper_2210_09147_b200 import engine, model as mdl, streams
    c5 = [1024, 2048, 4096, 8192, 8192, 4096, 2048, 1024] * 3 + [1024]
    cases = [("C2_adam", "C2 (32-layer 2048-wide, batch 1, D=1) with Adam", [2048] * 33, 1, True, 1, 32,
              "adam", "mse"),
             ("C3", "64-layer 4096-wide MLP inference wave, D=8 stages on 1 GPU", [4096] * 65, 8, False, 1, 8,
              "sgd", "mse"),
             ("C4", "32-layer 4096-wide MLP, micro-batch 16, D=8 stages on 1 GPU", [4096] * 33, 8, True, 16, 8,
              "sgd", "mse"),
             ("C4_adam_ce", "C4 with Adam and softmax-CE (PAPER.md:863 replay batches use Adam), D=8 on 1 GPU",
              [4096] * 33, 8, True, 16, 8, "adam", "softmax_ce"),
             ("C4_m32", "C4's network with micro-batch 32 (replay window 32, SPEC.md:463), D=8 on 1 GPU",
              [4096] * 33, 8, True, 32, 8, "sgd", "mse"),
             ("C5", "uneven widths 1024..8192 (24 layers), D=8 stages on 1 GPU", c5, 8, True, 1, 16, "sgd", "mse")]
    res = {}
    for name, desc, widths, D, learn, M, ticks, opt, loss in cases:
        try:
            m = mdl.mlp(widths, seed=0, dtype=np.float32, loss=loss)
            st = streams.SmoothStream(widths[0], widths[-1], seed=1, batch=M)
            xs, ys = st.block(0, ticks)
            if loss == "softmax_ce":
                ys = np.argmax(ys, axis=-1).astype(np.float32)
            xs = torch.tensor(xs, dtype=torch.float32, device="cuda")
            ys = torch.tensor(ys, dtype=torch.float32, device="cuda")
            x0 = xs[0].cpu().numpy() if M > 1 else xs[0, 0].cpu().numpy()
            y0 = ys[0].cpu().numpy() if M > 1 else ys[0, 0].cpu().numpy()
            p = engine.Pipeline(m, balanced_counts(widths, D, learn), opt, (1e-3 if opt == "sgd" else 1e-4)
                                if learn else 0.0, x0, y0, learn=learn)
            # untimed runs until every stage is past its warm-up gate (t >= 2D - h - 1):
            # before it a stage neither updates nor writes its weights back
            for _ in range(-(-(2 * D - 1) // ticks)):
                p.run(xs, ys)
            best = 1e30
            for _ in range(3):
                p.run(xs, ys)
                p.sync()
                best = min(best, p.last_kernel_ms())
            us = best * 1e3 / ticks
            byt = algorithmic_bytes_per_tick(widths, learn, opt)
            res[name] = {"workload": desc, "kernel": KERNEL_NAMES[p.kernel_path], "tick_us": round(us, 1), "samples_per_s": round(M * 1e6 / us, 1),
                         "achieved_gbs": round(byt / (us * 1e-6) / 1e9, 1),
                         "frac_of_hbm_roofline": round(byt / (us * 1e-6) / 1e9 / peak, 4)}
            p.close()
            del xs, ys
            torch.cuda.empty_cache()
        except Exception as e:  # report, do not hide
            res[name] = {"workload": desc, "error": repr(e)[:200]}
    return res


KERNEL_NAMES = {"panel": "pt::panel_kernel", "tile": "pt::tile_kernel (tcgen05)", "tick": "pt::tick_kernel"}


def load_traffic(path_kind="panel"):
    """dram bytes per tick of the bench kernel from the committed ncu capture, if any."""
    path = os.path.join(ROOT, "profiles", f"ncu_{path_kind}_kernel.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get("dram_bytes_per_tick"), d
    except Exception:
        return None, None


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist

    from paper_2210_09147_b200 import engine, model as mdl, streams

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        if os.environ.get("PT_BENCH_ONE_DEVICE"):
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        gloo = dist.new_group(backend="gloo")
    D = max(world, 1)
    widths = [args.width] * (args.layers + 1)
    counts = plan_counts(args.layers, D)
    m = mdl.mlp(widths, seed=0, dtype=np.float32)
    st = streams.SmoothStream(widths[0], widths[-1], seed=1)
    T = args.ticks
    xs_h, ys_h = st.block(0, T)
    xs_h, ys_h = xs_h.astype(np.float32), ys_h.astype(np.float32)
    dev = torch.device("cuda", local)
    if world > 1:
        from paper_2210_09147_b200 import dist as pdist
        pipe = pdist.build_distributed(m, counts, "sgd", 1e-3, xs_h[0, 0], ys_h[0, 0], group=gloo)
    else:
        pipe = engine.Pipeline(m, counts, "sgd", 1e-3, xs_h[0, 0], ys_h[0, 0])
    first = pipe.local_first == 0
    last = pipe.local_first + pipe.local_count == pipe.D
    xs = torch.from_numpy(xs_h).to(dev) if first else None
    ys = torch.from_numpy(ys_h).to(dev) if last else None
    stream = torch.cuda.Stream(device=dev)  # the library launches on this stream; events too
    pipe.set_stream(stream)
    local_widths = widths[pipe.sfl[pipe.local_first]:pipe.sfl[pipe.local_first + pipe.local_count] + 1]
    bytes_tick = algorithmic_bytes_per_tick(local_widths, True)
    weights_bytes = sum(4 * local_widths[i] * local_widths[i + 1] for i in range(len(local_widths) - 1))
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    flush = weights_bytes < 2 * l2
    flush_buf = torch.empty(2 * l2 // 4, dtype=torch.float32, device=dev) if flush else None

    def barrier():
        if world > 1:
            dist.barrier(gloo)

    # warm-up (inputs were produced on the default stream)
    torch.cuda.synchronize()
    for _ in range(args.warmup):
        pipe.run(xs, ys, T)
    pipe.sync()
    torch.cuda.synchronize()

    # timed region: K steps, device time on the library's stream (= torch's current stream)
    sampler = ClockSampler(local)
    sampler.start()
    kernel_ms = []
    barrier()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * args.steps)]
    for k in range(args.steps):
        if flush:
            with torch.cuda.stream(stream):
                flush_buf.fill_(float(k))
        ev[2 * k].record(stream)
        pipe.run(xs, ys, T)
        ev[2 * k + 1].record(stream)
        kernel_ms.append(None)
    torch.cuda.synchronize()
    pipe.sync()
    step_ms = [ev[2 * k].elapsed_time(ev[2 * k + 1]) for k in range(args.steps)]
    barrier()
    clocks = sampler.stop()
    # per-launch duration of the tick kernel alone (library events around the launch)
    pipe.run(xs, ys, T)
    pipe.sync()
    launch_ms = pipe.last_kernel_ms()
    launch_ms_local = launch_ms
    total_ms = sum(step_ms)
    if world > 1:
        t = torch.tensor([total_ms, launch_ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=gloo)
        total_ms, launch_ms = float(t[0]), float(t[1])
    samples = args.steps * T * BATCH
    value = samples / (total_ms / 1e3)

    # e2e: the public per-run API with pinned host buffers (H2D in, D2H out, synchronous)
    xs_pin = torch.from_numpy(xs_h).pin_memory() if first else None
    ys_pin = torch.from_numpy(ys_h).pin_memory() if last else None
    e2e_steps = max(3, args.steps // 2)
    pipe.set_stream(None)
    pipe.run(xs_pin.numpy() if first else None, ys_pin.numpy() if last else None, T) if (first or last) else None
    barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        if first or last:
            pipe.run(xs_pin.numpy() if first else None, ys_pin.numpy() if last else None, T)
        else:
            pipe.run(None, None, T)
            pipe.sync()
    e2e_s = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([e2e_s], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=gloo)
        e2e_s = float(t[0])
    e2e_value = e2e_steps * T * BATCH / e2e_s
    # the per-sample drop-in path (SURVEY.md §8(d) "two API paths"): Pipeline.step -> pt_step,
    # host buffers, one synchronous tick per call (H2D x and y, tick, D2H output and loss)
    step_api = None
    if world == 1:
        for t in range(8):
            pipe.step(xs_h[t % T, 0], ys_h[t % T, 0])
        n_calls = 64
        t0 = time.perf_counter()
        for t in range(n_calls):
            pipe.step(xs_h[t % T, 0], ys_h[t % T, 0])
        el = time.perf_counter() - t0
        step_api = {"value": round(n_calls / el, 2), "unit": "samples/s", "us_per_call": round(el / n_calls * 1e6, 2),
                    "api": "engine.Pipeline.step -> pt_step (host buffers, one synchronous tick per call)"}
    # per-rank (per-stage) roofline: each rank's own launch time over its own stage's bytes
    peak_r = None
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peak_r = float(json.load(f)["hbm_gbs"])
    except Exception:
        peak_r = 6650.0
    mine = {"rank": rank, "stages": [pipe.local_first + 1, pipe.local_first + pipe.local_count],
            "kernel": KERNEL_NAMES[pipe.kernel_path], "launch_ms": round(launch_ms_local, 4),
            "algorithmic_bytes_per_launch": bytes_tick * T,
            "achieved_gbs": round(bytes_tick * T / (launch_ms_local / 1e3) / 1e9, 1),
            "frac": round(bytes_tick * T / (launch_ms_local / 1e3) / 1e9 / peak_r, 4)}
    per_rank = [mine]
    if world > 1:
        per_rank = [None] * world
        dist.all_gather_object(per_rank, mine, group=gloo)
    kpath = pipe.kernel_path
    pipe.close()  # ends the per-sample API's resident launch before other pipelines run
    h2d = T * BATCH * (widths[0] + widths[-1]) * 4
    d2h = T * BATCH * widths[-1] * 4 + T * 4 + T

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    achieved = bytes_tick * T / (launch_ms / 1e3) / 1e9
    peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(peaks_path) as f:
            peak, peak_src = float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        peak, peak_src = 6650.0, "fallback (B200_PROFILING.md)"
    tpt, ncu = load_traffic(kpath)
    if ncu is None or ncu.get("config") != {"width": args.width, "layers": args.layers, "stages": D}:
        tpt = None  # the committed capture is for another workload
    roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4), "traffic": (tpt * T if tpt else None),
            "kernel": KERNEL_NAMES[kpath], "algorithmic_bytes_per_launch": bytes_tick * T,
            "launch_ms": round(launch_ms, 4), "peak_source": peak_src}
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        v, cores, sample, _ = cpu_reference(widths, 1, args.cpu_seconds)
        cpu = {"value": round(v, 4), "unit": "samples/s", "cores": cores, "kind": "port", "sample": sample}
    extra = None
    if world == 1 and not args.no_extra:
        extra = extra_configs(peak)
    out = {
        "metric": METRIC, "value": round(value, 2), "unit": "samples/s", "n_gpus": max(world, args.gpus if world == 1 else world),
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(total_ms / args.steps, 4),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "fp32",
        "data": "synthetic smooth-d stream (SURVEY.md §8(d)), random-init weights (SPEC.md:106)",
        "config": {"workload": f"C2: {args.layers}-layer {args.width}-wide ReLU MLP, online learning, batch 1, "
                               f"D={D} stage(s), one stage per GPU",
                   "model": f"mlp-{args.layers}x{args.width}", "global_batch": BATCH, "seq_len": 1,
                   "parallelism": f"pp{D}", "ticks_per_step": T,
                   "l2": ("flushed between steps" if flush else "weights per GPU exceed L2 (inputs larger than L2)")},
        "latency": {"tick_us": round(1e3 * total_ms / (args.steps * T), 2),
                    "sample_latency_ticks": D, "sample_latency_us": round(1e3 * total_ms / (args.steps * T) * D, 2)},
        "roofline": roof,
        "per_rank": per_rank,
        "cpu_baseline": cpu,
        # job-wide bytes: xs enter at stage 1's GPU, targets and results at stage D's
        "e2e": {"value": round(e2e_value, 2), "unit": "samples/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h},
        "step_api": step_api,
        "gpu_launches": 2 * args.steps,
        "clocks": clocks,
        "other_configs": extra,
    }
    print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
