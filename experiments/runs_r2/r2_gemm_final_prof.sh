#!/bin/bash
# ncu --set full of the final CTA-pair GEMM launches of one C3 epoch (bench command)
cd $GRAFT_REPO_ROOT 2>/dev/null || true
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --hoisted 0 --coresident 0"
$CMD > /dev/null 2>&1; echo plain rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:gemm_tf32 -s 5 -c 5 -o gpurun_out/gemm_C3_final $CMD > gpurun_out/gemm_final_ncu.log 2>&1; echo ncu rc=$?
