#!/bin/bash
# loss kernel with 8 lanes per row: parity (epoch + edge-case tests) and its launch times
cd $GRAFT_REPO_ROOT 2>/dev/null || true
python -m pytest tests/test_gpu_epoch.py tests/test_gpu_edge_cases.py -x -q > gpurun_out/loss_pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/loss_pytest.log
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/loss_bench.json 2>gpurun_out/loss_bench.err; echo bench rc=$?; cut -c1-300 gpurun_out/loss_bench.json
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:loss_kernel -c 6 --csv --log-file gpurun_out/loss_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --hoisted 0 --coresident 0 > /dev/null 2>&1; echo ncu rc=$?
grep loss_kernel gpurun_out/loss_launches.csv | awk -F'","' '{print $NF}'
