#!/bin/bash
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --hoisted 0"
timeout 300 $B > gpurun_out/fx_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --kernel-name-base demangled -k regex:"gemm_tf32_kernel<.bool.1" -s 1 -c 1 -o gpurun_out/fx_wgrad_mn $B > gpurun_out/fx_ncu.log 2>&1
STEPS=5 bash tools/ablation.sh 4 C4:cache_int8 C5:cache_int8 > gpurun_out/fx_abl.log 2>&1
