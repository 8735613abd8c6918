#!/bin/bash
# ncu --set full of the C3 p=1 SpMM launches (256- and 44-wide) after a clean run of the same command
cd $GRAFT_REPO_ROOT 2>/dev/null || true
CMD="python tools/spmm_bench.py --config C3 --p 1 --variants shape:3 --widths 256,44 --reps 1"
$CMD > gpurun_out/np_plain.log 2>&1; echo plain rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:spmm_kernel -s 2 -c 3 -o gpurun_out/spmm_c3_narrow $CMD > gpurun_out/np_ncu.log 2>&1; echo ncu rc=$?
