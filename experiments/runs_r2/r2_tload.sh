#!/bin/bash
cd $GRAFT_REPO_ROOT 2>/dev/null || true
timeout 900 python tools/spmm_bench.py --config C3 --p 1 --variants "tload:0;tload:1;tload:2;tload:0" --widths 256,44 --reps 7 2>&1 | grep '{'
timeout 900 python tools/spmm_bench.py --config C4 --p 1 --variants "tload:0;tload:1;tload:2" --widths 256 --reps 5 2>&1 | grep '{'
timeout 1700 python -m pytest tests/test_gpu_epoch.py -q -p no:cacheprovider -k "C4_C5 or fixed_eps" 2>&1 | tail -5
