#!/bin/bash
# narrow SpMM with __launch_bounds__(256, 5) (48 regs, small spill) vs default (61 regs, 4 blocks/SM)
cd $GRAFT_REPO_ROOT 2>/dev/null || true
for v in base minb5 base minb5; do
  cp _ab/libcdfgnn_$v.so paper_2408_00232_b200/libcdfgnn.so
  timeout 600 python tools/spmm_bench.py --config C3 --p 1 --variants "shape:3" --widths 44 --reps 15 2>&1 | grep '{' | sed "s/^/$v /"
  timeout 600 python tools/spmm_bench.py --config C4 --p 1 --variants "shape:3" --widths 48 --reps 9 2>&1 | grep '{' | sed "s/^/$v /"
done
cp _ab/libcdfgnn_base.so paper_2408_00232_b200/libcdfgnn.so
