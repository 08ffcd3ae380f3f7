"""bench.py keeps the driver's JSON contract: the reference arm here (CPU), the GPU arm on a
B200 (a short run)."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    out = _run(["--impl", "reference", "--steps", "1", "--warmup", "3"], 300)
    assert out["impl"] == "reference" and out["unit"] == "samples/s" and out["value"] > 0
    assert out["higher_is_better"] is True and out["cpu_baseline"]["kind"] in ("port", "reference")
    assert out["e2e"]["h2d_bytes_per_step"] == 0 and out["e2e"]["value"] == out["value"]


@pytest.mark.gpu
def test_gpu_arm_line():
    out = _run(["--steps", "2", "--warmup", "3", "--ticks", "8", "--no-extra", "--no-cpu-baseline"], 600)
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks", "step_api"):
        assert k in out, k
    assert out["n_gpus"] == 1 and out["steps"] == 2 and out["warmup"] == 3 and out["value"] > 0
    assert out["roofline"]["bound"] == "hbm" and 0 < out["roofline"]["frac"] < 1
    assert out["e2e"]["h2d_bytes_per_step"] > 0 and out["e2e"]["d2h_bytes_per_step"] > 0
    assert out["gpu_launches"] > 0 and out["step_api"]["value"] > 0
    assert "workload" in out["config"]


@pytest.mark.gpu
def test_gpu_arm_two_ranks_one_device():
    """The multi-GPU launch path (torchrun, one stage per rank, CUDA IPC exchange), with both
    ranks on GPU 0 (PT_BENCH_ONE_DEVICE; time-sliced, so the number itself is meaningless):
    rank 0 prints one line for the whole job."""
    env = dict(os.environ, PT_BENCH_ONE_DEVICE="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29531", os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "2", "--warmup", "3", "--ticks", "8", "--no-extra"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    out = json.loads(lines[0])
    assert out["n_gpus"] == 2 and out["config"]["parallelism"] == "pp2" and out["value"] > 0
    assert out["latency"]["sample_latency_ticks"] == 2
