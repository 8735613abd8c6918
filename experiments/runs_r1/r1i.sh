#!/bin/bash
set -x
timeout 900 python tools/spmm_bench.py --config C3 --p 1 --widths 44 --variants ";chunk:1024;chunk:4096;chunk:0;chunk:512" 2>&1 | grep "{" > gpurun_out/r1i_chunk_p1.jsonl
timeout 900 python tools/spmm_bench.py --config C3 --p 4 --widths 44 --variants ";chunk:1024;chunk:4096;chunk:512" 2>&1 | grep "{" > gpurun_out/r1i_chunk_p4.jsonl
timeout 1500 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/r1i_pytest.log 2>&1; echo rc=$? >> gpurun_out/r1i_pytest.log
TR2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 900 $TR2 --master-port 29632 bench.py --gpus 2 --steps 10 --warmup 3 --hoisted 0 > gpurun_out/r1i_bench_n2.json 2> gpurun_out/r1i_bench_n2.err
