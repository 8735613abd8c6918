#!/bin/bash
# SpMM visiting order x vertex numbering at p = 4 (part 0, co-resident)
for rl in none classdeg; do
  timeout 900 python tools/spmm_bench.py --config C3 --p 4 --widths 256,44 --relabel $rl \
    --variants "order:0;order:1;order:2;order:2,heavy:1024;order:2,heavy:256" 2>&1 | grep "{" >> gpurun_out/order_exp4.jsonl
done
