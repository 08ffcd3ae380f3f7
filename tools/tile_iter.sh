#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -k tile -x -q > gpurun_out/pytest_tile.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tile.log
timeout 300 python tools/tile_trace.py > gpurun_out/tile_trace.log 2>&1
timeout 300 python -c "
import sys; sys.path.insert(0, 'tools')
from configs_probe import probe
probe('C4 32x4096 M=16', [4096] * 33, 1, M=16, ticks=4, reps=2)
probe('C4 32x4096 M=16 D=8 on 1 GPU', [4096] * 33, 8, M=16, ticks=8, reps=2)
" > gpurun_out/c4.log 2>&1
tail -3 gpurun_out/pytest_tile.log; cat gpurun_out/tile_trace.log; cat gpurun_out/c4.log
