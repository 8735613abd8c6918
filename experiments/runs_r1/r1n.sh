#!/bin/bash
TR2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
CDFGNN_DEV_BARRIER=1 timeout 900 $TR2 --master-port 29662 bench.py --gpus 2 --steps 10 --warmup 3 --hoisted 0 --no-e2e > gpurun_out/r1n_dev.json 2> gpurun_out/r1n_dev.err
timeout 900 $TR2 --master-port 29663 bench.py --gpus 2 --steps 10 --warmup 3 --hoisted 0 --no-e2e > gpurun_out/r1n_nccl.json 2> gpurun_out/r1n_nccl.err
B="python bench.py --config C4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --hoisted 0"
timeout 600 $B > gpurun_out/r1n_c4plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C4_p1.csv $B > gpurun_out/r1n_ncu.log 2>&1
