#!/bin/bash
# GEMM k-block 16 (64-B swizzle, 4 stages at N = 256) vs 32: parity first, then A/B epochs
cd $GRAFT_REPO_ROOT 2>/dev/null || true
cp _ab/libcdfgnn_bk16.so paper_2408_00232_b200/libcdfgnn.so
timeout 900 python -m pytest tests/test_gpu_gemm.py -x -q -p no:cacheprovider > gpurun_out/bk16_gemm_tests.log 2>&1; rc=$?; echo gemm tests rc=$rc; tail -3 gpurun_out/bk16_gemm_tests.log
if [ $rc -ne 0 ]; then exit 1; fi
for v in bk32 bk16 bk32 bk16; do
  cp _ab/libcdfgnn_$v.so paper_2408_00232_b200/libcdfgnn.so
  for C in C3 C4; do
    timeout 600 python bench.py --config $C --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --hoisted 0 --coresident 0 2>/dev/null | python -c "import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$v', '$C', d['value'], d['phase_ms']['gemm'], d['phase_ms']['spmm'])"
  done
done
cp _ab/libcdfgnn_bk16.so paper_2408_00232_b200/libcdfgnn.so
timeout 1500 python -m pytest tests/test_gpu_epoch.py tests/test_gpu_bench_config.py -x -q -p no:cacheprovider > gpurun_out/bk16_epoch_tests.log 2>&1; echo epoch tests rc=$?; tail -2 gpurun_out/bk16_epoch_tests.log
