#!/bin/bash
# Round-1 final profile pass (1 GPU): bench line, launch list, ncu --set full of the top kernels
# (wide + narrow SpMM, 3xTF32 GEMM) and of one co-resident C3 p=2 epoch's halo kernels.
# Every command runs once plainly (exit 0) before the same command runs under ncu.
set -x
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --hoisted 0"
H2="python tools/halo_bench.py --config C3 --p 2 --epochs 3"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
timeout 300 $B > gpurun_out/fplain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_launches_C3_p1.csv $B > gpurun_out/fncu_l.log 2>&1
timeout 300 $B > gpurun_out/fplain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"spmm_kernel<.int.32," -s 2 -c 1 -o gpurun_out/final_spmm_wide $B > gpurun_out/fncu_sw.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"spmm_kernel<.int.8," -s 2 -c 1 -o gpurun_out/final_spmm_narrow $B > gpurun_out/fncu_sn.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tf32 -s 3 -c 1 -o gpurun_out/final_gemm $B > gpurun_out/fncu_g.log 2>&1
timeout 300 $H2 > gpurun_out/fplain3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none -k regex:"gather_pack|master_kernel|mirror_apply|scatter_pack|put_kernel" -s 30 -c 20 -o gpurun_out/final_halo_C3_p2 $H2 > gpurun_out/fncu_h.log 2>&1
ls -la gpurun_out/
