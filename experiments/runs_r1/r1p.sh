#!/bin/bash
set -x
timeout 1500 python -m pytest tests/test_gpu_epoch.py tests/test_gpu_bench_config.py -x -q > gpurun_out/r1p_pytest.log 2>&1; echo rc=$? >> gpurun_out/r1p_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1p_smoke.log 2>&1; echo rc=$? >> gpurun_out/r1p_smoke.log
B="python bench.py --config C4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --hoisted 0"
timeout 600 $B > gpurun_out/r1p_c4plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C4_p1_c.csv -k regex:"loss|reduce_rows" $B > gpurun_out/r1p_ncu.log 2>&1
