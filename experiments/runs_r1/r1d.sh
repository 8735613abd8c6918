#!/bin/bash
# 2-GPU validation of the device NVLink barrier + scatter_pack unroll; bench at N=1 and N=2.
set -x
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 1500 python -m pytest tests/test_gpu_multi.py tests/test_gpu_halo.py -x -q > gpurun_out/r1d_pytest.log 2>&1; echo rc=$? >> gpurun_out/r1d_pytest.log
timeout 600 $TR --master-port 29601 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/r1d_bench_n2.json 2> gpurun_out/r1d_bench_n2.err
CDFGNN_NCCL_BARRIER=1 timeout 600 $TR --master-port 29602 bench.py --gpus 2 --steps 10 --warmup 3 --hoisted 0 > gpurun_out/r1d_bench_n2_ncclbar.json 2> gpurun_out/r1d_bench_n2_ncclbar.err
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r1d_bench_n1.json 2> gpurun_out/r1d_bench_n1.err
