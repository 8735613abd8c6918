#!/bin/bash
for v in "0 0" "1 0" "1 1" "0 0" "1 0" "1 1"; do set -- $v; echo "overlap=$1 serial=$2"; CDFGNN_OVL_SERIAL=$2 timeout 300 python tools/halo_bench.py --config C3 --p 2 --epochs 4 --overlap $1 | tail -1; done
