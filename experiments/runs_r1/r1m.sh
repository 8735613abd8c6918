#!/bin/bash
bash tools/scale.sh 4 10 cache_int8 > gpurun_out/r1m_scale.log 2>&1
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --hoisted 0"
timeout 300 $B > gpurun_out/r1m_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"spmm_kernel<.int.32," -s 2 -c 1 -o gpurun_out/final_spmm_wide $B > gpurun_out/fncu_sw.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"spmm_kernel<.int.8," -s 2 -c 1 -o gpurun_out/final_spmm_narrow $B > gpurun_out/fncu_sn.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_launches_C3_p1.csv $B > gpurun_out/fncu_l.log 2>&1
