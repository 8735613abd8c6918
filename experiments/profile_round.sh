#!/bin/bash
# Round profile pass (1 GPU): bench line, launch list, ncu --set full of the top kernels.
# Every command runs once plainly (exit 0) before the same command runs under ncu.
set -x
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
H2="python tools/halo_bench.py --config C3 --p 2 --epochs 2"
H4="python tools/halo_bench.py --config C3 --p 4 --epochs 2"
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
timeout 300 $B > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C3_p1.csv $B > gpurun_out/ncu_l.log 2>&1
timeout 300 $B > gpurun_out/plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_kernel -s 4 -c 1 -o gpurun_out/spmm_C3_p1 $B > gpurun_out/ncu_s.log 2>&1
timeout 300 $B > gpurun_out/plain3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tf32 -s 5 -c 1 -o gpurun_out/gemm_C3_p1 $B > gpurun_out/ncu_g.log 2>&1
timeout 300 $H2 > gpurun_out/plain4.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:spmm_kernel --csv --log-file gpurun_out/spmm_C3_p2.csv $H2 > gpurun_out/ncu_h2.log 2>&1
timeout 300 $H4 > gpurun_out/plain5.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:spmm_kernel --csv --log-file gpurun_out/spmm_C3_p4.csv $H4 > gpurun_out/ncu_h4.log 2>&1
ls -la gpurun_out/
