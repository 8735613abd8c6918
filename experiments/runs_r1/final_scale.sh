#!/bin/bash
# Final C3 scaling on one 4-GPU box with the round's last code (N = 1, 2, 4) and the launch list.
bash tools/scale.sh 4 10 cache_int8 > gpurun_out/fsc_scale.log 2>&1
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --hoisted 0"
timeout 300 $B > gpurun_out/fsc_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fsc_launches_C3_p1.csv $B > gpurun_out/fsc_ncu.log 2>&1
