#!/bin/bash
# C4 at N = 1: launch list (GEMM shapes and times) after a clean run
cd $GRAFT_REPO_ROOT 2>/dev/null || true
CMD="python bench.py --config C4 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --hoisted 0 --coresident 0"
$CMD > gpurun_out/c4_plain.json 2> gpurun_out/c4_plain.err; echo plain rc=$?; cut -c1-300 gpurun_out/c4_plain.json
ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none -c 300 --csv --log-file gpurun_out/launches_C4_n1.csv $CMD > /dev/null 2>&1; echo ncu rc=$?
