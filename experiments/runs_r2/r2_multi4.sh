#!/bin/bash
cd $GRAFT_REPO_ROOT 2>/dev/null || true
timeout 2000 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider > gpurun_out/multi4.log 2>&1; tail -5 gpurun_out/multi4.log
