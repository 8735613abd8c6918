#!/bin/bash
# CTA pair only for BN >= 128 + warp-parallel split-K sum: parity, then epochs
cd $GRAFT_REPO_ROOT 2>/dev/null || true
timeout 300 python -m pytest tests/test_gpu_gemm.py -x -q -p no:cacheprovider > gpurun_out/pair2_gemm_tests.log 2>&1; rc=$?; echo gemm tests rc=$rc; tail -1 gpurun_out/pair2_gemm_tests.log
if [ $rc -ne 0 ]; then exit 1; fi
for r in 1 2; do
  for C in C3 C4; do
    timeout 400 python bench.py --config $C --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --hoisted 0 --coresident 0 2>/dev/null | python -c "import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$C', d['value'], d['phase_ms']['gemm'], d['phase_ms']['spmm'], d['clocks']['sm_mhz'])"
  done
done
timeout 1500 python -m pytest tests/test_gpu_epoch.py tests/test_gpu_bench_config.py tests/test_gpu_edge_cases.py -x -q -p no:cacheprovider > gpurun_out/pair2_epoch_tests.log 2>&1; echo epoch tests rc=$?; tail -1 gpurun_out/pair2_epoch_tests.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm_tf32|splitk" -c 12 --csv --log-file gpurun_out/pair2_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --hoisted 0 --coresident 0 > /dev/null 2>&1; echo ncu rc=$?
