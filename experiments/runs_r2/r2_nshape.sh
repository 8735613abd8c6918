#!/bin/bash
# narrow-row SpMM shapes: 8x2 UNR 8 (default, shape 3) vs 4x3 UNR 8 / 6 (shapes 7, 8), 4x3 UNR 4 (1)
cd $GRAFT_REPO_ROOT 2>/dev/null || true
V="shape:3;shape:7;shape:8;shape:1;shape:7,chunk:2048;shape:7,chunk:8192;shape:3"
timeout 900 python tools/spmm_bench.py --config C3 --p 1 --variants "$V" --widths 44 --reps 15 2>&1 | grep '{'
timeout 900 python tools/spmm_bench.py --config C3 --p 4 --variants "shape:3;shape:7;shape:8;shape:7,chunk:512;shape:3" --widths 44 --reps 15 2>&1 | grep '{'
timeout 900 python tools/spmm_bench.py --config C4 --p 1 --variants "shape:3;shape:7;shape:8;shape:3" --widths 48 --reps 9 2>&1 | grep '{'
timeout 900 python tools/spmm_bench.py --config C5 --p 1 --variants "shape:3;shape:7;shape:8;shape:3" --widths 48 --reps 9 2>&1 | grep '{'
