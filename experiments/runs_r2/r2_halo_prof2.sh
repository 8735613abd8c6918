#!/bin/bash
cd $GRAFT_REPO_ROOT 2>/dev/null || true
CMD="python tools/halo_bench.py --config C3 --p 4 --epochs 1"
$CMD > gpurun_out/halo_plain2.log 2>&1 && timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"gather_slot|master_slot|mirror_slot" -s 0 -c 12 -o gpurun_out/halo_prof_wide $CMD > gpurun_out/halo_ncu2.log 2>&1; echo ncu rc=$?
