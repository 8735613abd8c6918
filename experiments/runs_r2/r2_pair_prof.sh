#!/bin/bash
# ncu --set full of the CTA-pair GEMM (C3 T = X W0 launch) after a clean run
cd $GRAFT_REPO_ROOT 2>/dev/null || true
CMD="python bench.py --config C3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --hoisted 0 --coresident 0"
CDFGNN_GEMM_PAIR=1 $CMD > /dev/null 2>&1; echo plain rc=$?
CDFGNN_GEMM_PAIR=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tf32 -s 5 -c 1 -o gpurun_out/gemm_pair_C3 $CMD > gpurun_out/gemm_pair_ncu.log 2>&1; echo ncu rc=$?
