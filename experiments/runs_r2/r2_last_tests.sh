#!/bin/bash
# last full 1-GPU test run of the round
cd $GRAFT_REPO_ROOT 2>/dev/null || true
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_last.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/smoke_last.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_last.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_gpu_last.log
