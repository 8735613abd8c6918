#!/bin/bash
# SpMM visiting order x vertex numbering on the products-shaped graph (T >> L2)
for rl in none classdeg class; do
  timeout 1200 python tools/spmm_bench.py --config C4 --p 4 --widths 256,48 --relabel $rl \
    --variants "order:0;order:1;order:2,heavy:1024" 2>&1 | grep "{" >> gpurun_out/order_exp_c4.jsonl
done
