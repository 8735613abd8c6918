#!/bin/bash
# CTA-pair (cta_group::2) 3xTF32 GEMM: parity under CDFGNN_GEMM_PAIR=1, then A/B epochs
cd $GRAFT_REPO_ROOT 2>/dev/null || true
CDFGNN_GEMM_PAIR_VERBOSE=1 CDFGNN_GEMM_PAIR=1 timeout 300 python -m pytest tests/test_gpu_gemm.py -x -q -s -p no:cacheprovider > gpurun_out/pair_gemm_tests.log 2>&1; rc=$?; echo gemm tests rc=$rc; grep -m3 "co-resident\|passed\|failed" gpurun_out/pair_gemm_tests.log | cut -c1-300
if [ $rc -ne 0 ]; then exit 1; fi
for v in 0 1 0 1; do
  for C in C3 C4; do
    CDFGNN_GEMM_PAIR=$v timeout 400 python bench.py --config $C --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --hoisted 0 --coresident 0 2>/dev/null | python -c "import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('pair $v', '$C', d['value'], d['phase_ms']['gemm'], d['phase_ms']['spmm'], d['clocks']['sm_mhz'])"
  done
done
CDFGNN_GEMM_PAIR=1 timeout 900 python -m pytest tests/test_gpu_epoch.py tests/test_gpu_bench_config.py -x -q -p no:cacheprovider > gpurun_out/pair_epoch_tests.log 2>&1; echo epoch tests rc=$?; tail -2 gpurun_out/pair_epoch_tests.log
CMD="python bench.py --config C4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --hoisted 0 --coresident 0"
CDFGNN_GEMM_PAIR=1 timeout 900 ncu --metrics gpu__time_duration.sum,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed,l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed --clock-control none -k regex:gemm_tf32 -s 8 -c 8 --csv --log-file gpurun_out/pair_gemm_C4.csv $CMD > /dev/null 2>&1; echo ncu rc=$?
