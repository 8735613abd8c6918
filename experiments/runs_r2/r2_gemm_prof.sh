#!/bin/bash
# ncu --set full of one epoch's GEMMs (C4 and C3 at N = 1), after clean runs of the same commands
cd $GRAFT_REPO_ROOT 2>/dev/null || true
C4="python bench.py --config C4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --hoisted 0 --coresident 0"
C3="python bench.py --config C3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --hoisted 0 --coresident 0"
$C4 > gpurun_out/gp_c4.json 2>&1; echo c4 rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:gemm_tf32 -s 8 -c 8 -o gpurun_out/gemm_C4 $C4 > gpurun_out/gemm_C4_ncu.log 2>&1; echo ncu c4 rc=$?
$C3 > gpurun_out/gp_c3.json 2>&1; echo c3 rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:gemm_tf32 -s 5 -c 5 -o gpurun_out/gemm_C3 $C3 > gpurun_out/gemm_C3_ncu.log 2>&1; echo ncu c3 rc=$?
