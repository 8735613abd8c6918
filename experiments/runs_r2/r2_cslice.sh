#!/bin/bash
cd $GRAFT_REPO_ROOT 2>/dev/null || true
timeout 900 python tools/spmm_bench.py --config C3 --p 1 --variants "cslice:0;cslice:128;cslice:64;cslice:32" --widths 256 --reps 5 2>&1 | grep '{'
timeout 900 python tools/spmm_bench.py --config C3 --p 4 --variants "cslice:0;cslice:128;cslice:64" --widths 256 --reps 5 2>&1 | grep '{'
timeout 900 python tools/spmm_bench.py --config C4 --p 1 --variants "cslice:0;cslice:128;cslice:64" --widths 256 --reps 5 2>&1 | grep '{'
