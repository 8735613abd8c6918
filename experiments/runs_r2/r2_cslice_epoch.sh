#!/bin/bash
# in-epoch A/B of column-sliced wide SpMM (T slices that fit L2: less DRAM traffic, less power)
cd $GRAFT_REPO_ROOT 2>/dev/null || true
for v in 0 128 0 128 64; do
  CDFGNN_SPMM_CSLICE=$v timeout 600 python bench.py --config C3 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --hoisted 0 --coresident 0 2>/dev/null | python -c "import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('cslice $v', d['value'], d['phase_ms']['spmm'], d['clocks'], d['roofline']['dram_gbs'])"
done
