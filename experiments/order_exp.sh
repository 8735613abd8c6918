#!/bin/bash
# SpMM visiting order x vertex numbering experiment (C3, p = 1).
for rl in none class classdeg; do
  timeout 900 python tools/spmm_bench.py --config C3 --p 1 --widths 256,44 --relabel $rl \
    --variants "order:0;order:1;order:2;order:2,heavy:1024" 2>&1 | grep "{" >> gpurun_out/order_exp.jsonl
done
