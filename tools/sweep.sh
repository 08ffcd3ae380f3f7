python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
python tools/trace_probe.py one | grep -E "^==|->" | head -8
