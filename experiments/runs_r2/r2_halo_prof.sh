#!/bin/bash
cd $GRAFT_REPO_ROOT 2>/dev/null || true
timeout 1200 python -m pytest tests/test_gpu_halo.py tests/test_gpu_epoch.py -q -x -p no:cacheprovider > gpurun_out/halo_tests.log 2>&1; tail -3 gpurun_out/halo_tests.log
CMD="python tools/halo_bench.py --config C3 --p 4 --epochs 2"
$CMD > gpurun_out/halo_plain.log 2>&1 && timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"gather_slot|master_slot|mirror_slot" -s 12 -c 6 -o gpurun_out/halo_prof $CMD > gpurun_out/halo_ncu.log 2>&1; echo ncu rc=$?
tail -2 gpurun_out/halo_plain.log
