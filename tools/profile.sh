#!/bin/bash
# Round profiling recipe (B200_PROFILING.md): launch list + one full capture of the tick kernel.
set -x
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --ticks 16 --no-cpu-baseline > gpurun_out/launches_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:tick_kernel -s 1 -c 1 -f -o gpurun_out/prof_tick \
    python bench.py --steps 1 --warmup 1 --ticks 8 --no-cpu-baseline > gpurun_out/prof_bench.log 2>&1
ls -la gpurun_out
