#!/bin/bash
set -x
timeout 1500 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_epoch.py tests/test_gpu_bench_config.py -x -q > gpurun_out/r1o_pytest.log 2>&1; echo rc=$? >> gpurun_out/r1o_pytest.log
B="python bench.py --config C4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --hoisted 0"
timeout 600 $B > gpurun_out/r1o_c4plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_C4_p1_b.csv -k regex:transpose $B > gpurun_out/r1o_ncu.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r1o_bench_n1.json 2> gpurun_out/r1o_bench_n1.err
