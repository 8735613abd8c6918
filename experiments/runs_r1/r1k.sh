#!/bin/bash
set -x
timeout 1500 python -m pytest tests/test_gpu_halo.py tests/test_gpu_epoch.py tests/test_gpu_multi.py -x -q > gpurun_out/r1k_pytest.log 2>&1; echo rc=$? >> gpurun_out/r1k_pytest.log
H2="python tools/halo_bench.py --config C3 --p 2 --epochs 3"
timeout 300 $H2 > gpurun_out/r1k_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none -k regex:"master" -s 12 -c 8 -o gpurun_out/r1k_halo $H2 > gpurun_out/r1k_ncu.log 2>&1
CDFGNN_MASTER_CP=0 timeout 300 $H2 > gpurun_out/r1k_plain_nocp.log 2>&1
STEPS=5 bash tools/ablation.sh 2 C4:cache_int8 > gpurun_out/r1k_abl.log 2>&1
