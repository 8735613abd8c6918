#!/bin/bash
set -x
timeout 900 python -m pytest tests/test_gpu_epoch.py -x -q -k "pipelined or hoisted" > gpurun_out/r1f_pytest.log 2>&1; echo rc=$? >> gpurun_out/r1f_pytest.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r1f_bench_n1.json 2> gpurun_out/r1f_bench_n1.err
TR2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 900 $TR2 --master-port 29622 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/r1f_bench_n2.json 2> gpurun_out/r1f_bench_n2.err
