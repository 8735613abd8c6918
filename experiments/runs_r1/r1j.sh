#!/bin/bash
set -x
timeout 1500 python -m pytest tests/test_gpu_halo.py tests/test_gpu_epoch.py tests/test_gpu_multi.py -x -q > gpurun_out/r1j_pytest.log 2>&1; echo rc=$? >> gpurun_out/r1j_pytest.log
H2="python tools/halo_bench.py --config C3 --p 2 --epochs 3"
timeout 300 $H2 > gpurun_out/r1j_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none -k regex:"master_kernel|map_copy" -s 12 -c 8 -o gpurun_out/r1j_halo $H2 > gpurun_out/r1j_ncu.log 2>&1
STEPS=5 bash tools/ablation.sh 1 C4:cache_int8 > gpurun_out/r1j_abl.log 2>&1
STEPS=5 bash tools/ablation.sh 2 C4:cache_int8 >> gpurun_out/r1j_abl.log 2>&1
TR2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 900 $TR2 --master-port 29642 bench.py --gpus 2 --steps 10 --warmup 3 --hoisted 0 > gpurun_out/r1j_bench_n2.json 2> gpurun_out/r1j_bench_n2.err
