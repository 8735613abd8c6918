#!/bin/bash
# Halo kernels after the receive-table / code-row / narrow-shape changes: GPU halo+epoch tests,
# co-resident C3 p=2 phase times, ncu --set full of one epoch's halo launches.
set -x
timeout 900 python -m pytest tests/test_gpu_halo.py tests/test_gpu_epoch.py -x -q > gpurun_out/h2_pytest.log 2>&1; echo rc=$? >> gpurun_out/h2_pytest.log
H2="python tools/halo_bench.py --config C3 --p 2 --epochs 4"
timeout 300 $H2 > gpurun_out/h2b_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gather_pack|master_kernel|mirror_apply|scatter_pack" -s 30 -c 20 -o gpurun_out/halo2_C3_p2 python tools/halo_bench.py --config C3 --p 2 --epochs 3 > gpurun_out/ncu_halo2.log 2>&1
ls -la gpurun_out/
