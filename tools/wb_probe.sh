mkdir -p gpurun_out
PT_WB=1 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
PT_WB=1 timeout 300 python tools/trace_probe.py one 2>&1 | head -14
PT_WB=1 timeout 300 python tools/configs_probe.py 2>&1 | head -4
timeout 300 python tools/configs_probe.py 2>&1 | head -3
