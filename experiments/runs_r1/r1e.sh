#!/bin/bash
# SpMM shape sweep (C3 p=1, p=4 part 0) and N=4 bench.
set -x
timeout 900 python tools/spmm_bench.py --config C3 --p 1 --widths 256,44 --variants ";shape:0;shape:4;shape:5;shape:6;wshape:1;wshape:2;wshape:3;unr:2;unr:8" 2>&1 | grep "{" > gpurun_out/sweep_p1.jsonl
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 900 $TR --master-port 29611 bench.py --gpus 4 --steps 10 --warmup 3 > gpurun_out/r1e_bench_n4.json 2> gpurun_out/r1e_bench_n4.err
TR2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 900 $TR2 --master-port 29612 bench.py --gpus 2 --steps 10 --warmup 3 --hoisted 0 > gpurun_out/r1e_bench_n2.json 2> gpurun_out/r1e_bench_n2.err
