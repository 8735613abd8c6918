#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_epoch.py tests/test_gpu_spmm.py -x -q > gpurun_out/r1c_pytest.log 2>&1; echo rc=$? >> gpurun_out/r1c_pytest.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r1c_bench.json 2> gpurun_out/r1c_bench.err
bash tools/order_exp.sh
