#!/bin/bash
timeout 400 python tools/spmm_bench.py --config C3 --p 1 --panels 256 --widths 256,44 --variants "hint:0;hint:1;hint:2" 2>&1 | grep "{"
for h in 0 1 2; do
  for o in 1 0; do echo "hint=$h overlap=$o"; CDFGNN_SPMM_HINT=$h timeout 300 python tools/halo_bench.py --config C3 --p 2 --epochs 3 --overlap $o | tail -1; done
done
