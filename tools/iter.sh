#!/bin/bash
# quick iteration on one GPU: parity tests, phase trace, config probe
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/trace_probe.py one > gpurun_out/trace.log 2>&1
timeout 600 python tools/configs_probe.py > gpurun_out/configs.log 2>&1
PT_SLOT_KB=32 timeout 600 python tools/configs_probe.py > gpurun_out/configs32.log 2>&1
tail -3 gpurun_out/pytest_gpu.log; head -14 gpurun_out/trace.log; cat gpurun_out/configs.log; echo "--- 32K:"; cat gpurun_out/configs32.log
