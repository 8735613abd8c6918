#!/bin/bash
cd $GRAFT_REPO_ROOT 2>/dev/null || true
timeout 900 python tools/spmm_bench.py --config C3 --p 1 --variants "chunk:0" --widths 256,44 --reps 7 2>&1 | grep '{'
