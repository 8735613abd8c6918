#!/bin/bash
cd $GRAFT_REPO_ROOT 2>/dev/null || true
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r2.json 2> gpurun_out/bench_r2.err; echo bench rc=$?
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --hoisted 0"
$CMD > gpurun_out/bench_small.json 2> gpurun_out/bench_small.err && ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_r2.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo ncu rc=$?
