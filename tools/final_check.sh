#!/bin/bash
# End-of-round measurement: the profiling recipe, a one-device two-rank bench smoke, and the
# per-GPU stage-share proxy for the scaling run.
bash tools/profile.sh
PT_BENCH_ONE_DEVICE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 2 --warmup 3 --no-extra \
    > gpurun_out/bench_n2_onedevice.json 2> gpurun_out/bench_n2_onedevice.err
timeout 600 python tools/scale_proxy.py > gpurun_out/scale_proxy.log 2>&1
cat gpurun_out/bench_n2_onedevice.json; tail -3 gpurun_out/bench_n2_onedevice.err; cat gpurun_out/scale_proxy.log
