#!/bin/bash
# 3xTF32 converter variants: bk16 (generic ld/st), bk16s (explicit shared ld/st), bk16sb (+ pre-split
# weight lo parts, converters split A only): parity of the last, then A/B epochs
cd $GRAFT_REPO_ROOT 2>/dev/null || true
cp _ab/libcdfgnn_bk16sb.so paper_2408_00232_b200/libcdfgnn.so
timeout 900 python -m pytest tests/test_gpu_gemm.py -x -q -p no:cacheprovider > gpurun_out/blo_gemm_tests.log 2>&1; rc=$?; echo gemm tests rc=$rc; tail -3 gpurun_out/blo_gemm_tests.log
if [ $rc -ne 0 ]; then exit 1; fi
for v in bk16 bk16s bk16sb bk16 bk16s bk16sb; do
  cp _ab/libcdfgnn_$v.so paper_2408_00232_b200/libcdfgnn.so
  for C in C3 C4; do
    timeout 600 python bench.py --config $C --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --hoisted 0 --coresident 0 2>/dev/null | python -c "import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$v', '$C', d['value'], d['phase_ms']['gemm'], d['phase_ms']['spmm'])"
  done
done
cp _ab/libcdfgnn_bk16sb.so paper_2408_00232_b200/libcdfgnn.so
timeout 1500 python -m pytest tests/test_gpu_epoch.py tests/test_gpu_bench_config.py -x -q -p no:cacheprovider > gpurun_out/blo_epoch_tests.log 2>&1; echo epoch tests rc=$?; tail -2 gpurun_out/blo_epoch_tests.log
CMD="python bench.py --config C4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --hoisted 0 --coresident 0"
timeout 1200 ncu --metrics gpu__time_duration.sum,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed,l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed --clock-control none -k regex:gemm_tf32 -s 8 -c 8 --csv --log-file gpurun_out/blo_gemm_C4.csv $CMD > /dev/null 2>&1; echo ncu rc=$?
