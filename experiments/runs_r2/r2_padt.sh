#!/bin/bash
# SpMM operand rows padded to 128-byte lines (CDFGNN_SPMM_PADT, default on) vs off: parity, then A/B
cd $GRAFT_REPO_ROOT 2>/dev/null || true
timeout 1800 python -m pytest tests/test_gpu_epoch.py tests/test_gpu_bench_config.py tests/test_gpu_spmm.py tests/test_gpu_edge_cases.py tests/test_gpu_coresident_c3.py -x -q -p no:cacheprovider > gpurun_out/padt_tests.log 2>&1; rc=$?; echo tests rc=$rc; tail -2 gpurun_out/padt_tests.log
if [ $rc -ne 0 ]; then exit 1; fi
for v in 0 1 0 1; do
  for C in C3 C4; do
    CDFGNN_SPMM_PADT=$v timeout 600 python bench.py --config $C --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --hoisted 0 --coresident $([ $C = C3 ] && echo 4 || echo 0) 2>/dev/null | python -c "import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('padt $v', '$C', d['value'], d['phase_ms']['gemm'], d['phase_ms']['spmm'], (d.get('coresident_p4') or {}).get('value'), d['clocks']['sm_mhz'])"
  done
done
CDFGNN_SPMM_PADT=1 timeout 900 ncu --metrics gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:spmm_kernel -c 8 --csv --log-file gpurun_out/padt_spmm.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --hoisted 0 --coresident 0 > /dev/null 2>&1; echo ncu rc=$?
