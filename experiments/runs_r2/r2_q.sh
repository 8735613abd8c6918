#!/bin/bash
cd $GRAFT_REPO_ROOT 2>/dev/null || true
timeout 1200 python -m pytest tests/test_gpu_halo.py tests/test_gpu_epoch.py -q -x -p no:cacheprovider > gpurun_out/q_tests.log 2>&1; tail -3 gpurun_out/q_tests.log
timeout 900 python tools/halo_bench.py --config C3 --p 4 --epochs 4 > gpurun_out/halo_c3p4_q.log 2>&1; tail -2 gpurun_out/halo_c3p4_q.log
timeout 900 python tools/halo_bench.py --config C4 --p 4 --epochs 4 > gpurun_out/halo_c4p4_q.log 2>&1; tail -2 gpurun_out/halo_c4p4_q.log
