#!/bin/bash
cd $GRAFT_REPO_ROOT 2>/dev/null || true
timeout 2000 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/fuse_tests.log 2>&1; tail -3 gpurun_out/fuse_tests.log
timeout 900 python tools/halo_bench.py --config C3 --p 4 --epochs 4 > gpurun_out/halo_c3p4_f.log 2>&1; tail -2 gpurun_out/halo_c3p4_f.log
timeout 900 python tools/halo_bench.py --config C4 --p 4 --epochs 4 > gpurun_out/halo_c4p4_f.log 2>&1; tail -2 gpurun_out/halo_c4p4_f.log
