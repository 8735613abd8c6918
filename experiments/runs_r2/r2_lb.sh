#!/bin/bash
cd $GRAFT_REPO_ROOT 2>/dev/null || true
for C in C3 C4; do timeout 900 python tools/halo_bench.py --config $C --p 4 --epochs 8 2>&1 | tail -2; done
