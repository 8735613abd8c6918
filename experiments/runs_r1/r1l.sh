#!/bin/bash
set -x
timeout 1500 python -m pytest tests/test_gpu_multi.py tests/test_gpu_epoch.py -x -q > gpurun_out/r1l_pytest.log 2>&1; echo rc=$? >> gpurun_out/r1l_pytest.log
TR2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 900 $TR2 --master-port 29652 bench.py --gpus 2 --steps 10 --warmup 3 --hoisted 0 > gpurun_out/r1l_bench_n2.json 2> gpurun_out/r1l_bench_n2.err
