#!/bin/bash
cd $GRAFT_REPO_ROOT 2>/dev/null || true
for rl in none class; do
timeout 900 python tools/spmm_bench.py --config C4 --p 1 --relabel $rl --variants "order:0;order:1;order:2" --widths 256,48 --reps 5 2>&1 | grep '{'
done
timeout 900 python tools/spmm_bench.py --config C3 --p 1 --relabel class --variants "order:0;order:1" --widths 256,44 --reps 5 2>&1 | grep '{'
