#!/bin/bash
# End-of-round check on a 4-GPU box: full GPU suite (multi-GPU tests at 4 ranks), smoke,
# C3 scaling N = 1, 2, 4, launch list of the N = 1 epoch.
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/f4_pytest.log 2>&1; echo rc=$? >> gpurun_out/f4_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f4_smoke.log 2>&1; echo rc=$? >> gpurun_out/f4_smoke.log
bash tools/scale.sh 4 10 cache_int8 > gpurun_out/f4_scale.log 2>&1
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --hoisted 0"
timeout 300 $B > gpurun_out/f4_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f4_launches_C3_p1.csv $B > gpurun_out/f4_ncu.log 2>&1
