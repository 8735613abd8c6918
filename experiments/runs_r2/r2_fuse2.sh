#!/bin/bash
cd $GRAFT_REPO_ROOT 2>/dev/null || true
for C in C3 C4; do for F in 0 1 0 1; do
timeout 900 python tools/halo_bench.py --config $C --p 4 --epochs 12 --fuse $F 2>&1 | tail -1
done; done
