#!/bin/bash
set -x
timeout 900 python -m pytest tests/test_gpu_halo.py tests/test_gpu_epoch.py tests/test_gpu_bench_config.py -x -q > gpurun_out/r1g_pytest.log 2>&1; echo rc=$? >> gpurun_out/r1g_pytest.log
H2="python tools/halo_bench.py --config C3 --p 2 --epochs 3"
timeout 300 $H2 > gpurun_out/r1g_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none -k regex:"gather_pack|master_kernel" -s 15 -c 12 -o gpurun_out/r1g_halo $H2 > gpurun_out/r1g_ncu.log 2>&1
