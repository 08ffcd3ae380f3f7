#!/bin/bash
# Round profiling recipe (B200_PROFILING.md): the bench line, a launch list of the bench
# command (PT_RESIDENT=0: ncu waits for every kernel to end, and a resident per-sample launch
# only ends when the host stops it), one full capture of the panel kernel (C2, the headline)
# and of the tile kernel (C4).
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
PT_RESIDENT=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --ticks 16 --no-cpu-baseline --no-extra > gpurun_out/launches_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:panel_kernel -s 3 -c 1 -f -o gpurun_out/prof_panel \
    python bench.py --steps 1 --warmup 3 --ticks 8 --no-cpu-baseline --no-extra > gpurun_out/prof_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tile_kernel -s 1 -c 1 -f -o gpurun_out/prof_tile \
    python tools/tile_one.py 8 > gpurun_out/prof_tile.log 2>&1
tail -3 gpurun_out/bench.err; ls -la gpurun_out
