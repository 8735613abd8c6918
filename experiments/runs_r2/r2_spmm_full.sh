#!/bin/bash
# ncu --set full of the bench command's first two SpMM launches (C3 p=1: 256- and 44-wide), final code
cd $GRAFT_REPO_ROOT 2>/dev/null || true
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --hoisted 0 --coresident 0"
$CMD > /dev/null 2>&1; echo plain rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:spmm_kernel -s 0 -c 2 -o gpurun_out/spmm_C3_p1_final $CMD > gpurun_out/spmm_full_ncu.log 2>&1; echo ncu rc=$?
