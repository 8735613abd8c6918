#!/bin/bash
# A/B: SpMM with the next CSR batch prefetched (pf) vs without (base)
cd $GRAFT_REPO_ROOT 2>/dev/null || true
for v in base pf base pf; do
  cp _ab/libcdfgnn_$v.so paper_2408_00232_b200/libcdfgnn.so
  echo "== $v"
  timeout 600 python tools/spmm_bench.py --config C3 --p 1 --variants "shape:3" --widths 256,44 --reps 7 2>&1 | grep '{'
  timeout 600 python tools/spmm_bench.py --config C3 --p 4 --variants "shape:3" --widths 256,44 --reps 7 2>&1 | grep '{'
  timeout 600 python tools/spmm_bench.py --config C4 --p 1 --variants "shape:3" --widths 256,48 --reps 5 2>&1 | grep '{'
done
cp _ab/libcdfgnn_pf.so paper_2408_00232_b200/libcdfgnn.so
timeout 1200 python -m pytest tests/test_gpu_spmm.py tests/test_gpu_bench_config.py -x -q 2>&1 | tail -2
