#!/bin/bash
cd $GRAFT_REPO_ROOT 2>/dev/null || true
CMD="python tools/halo_bench.py --config C3 --p 4 --epochs 1"
$CMD > gpurun_out/hp3_plain.log 2>&1 && timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"master_slot|gather_slot|mirror_slot" -s 0 -c 12 -o gpurun_out/halo_prof3 $CMD > gpurun_out/hp3_ncu.log 2>&1; echo ncu rc=$?
