#!/bin/bash
cd $GRAFT_REPO_ROOT 2>/dev/null || true
timeout 900 python -m pytest tests/test_gpu_spmm.py -q -x -p no:cacheprovider > gpurun_out/hub_tests.log 2>&1; tail -3 gpurun_out/hub_tests.log
timeout 900 python tools/spmm_bench.py --config C3 --p 1 --variants "hub:1;hub:0" --widths 256 --reps 5 > gpurun_out/hub_bench_p1.log 2>&1; cat gpurun_out/hub_bench_p1.log | grep '{'
timeout 900 python tools/spmm_bench.py --config C3 --p 4 --variants "hub:1;hub:0" --widths 256 --reps 5 > gpurun_out/hub_bench_p4.log 2>&1; cat gpurun_out/hub_bench_p4.log | grep '{'
CMD="python tools/spmm_bench.py --config C3 --p 1 --variants hub:1 --widths 256 --reps 1"
$CMD > gpurun_out/hub_plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_hub -c 1 -o gpurun_out/hub_prof2 $CMD > gpurun_out/hub_ncu.log 2>&1; echo ncu rc=$?
