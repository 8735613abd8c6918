#!/bin/bash
timeout 900 python tools/spmm_bench.py --config C3 --p 1 --widths 44 --variants ";unr:4;tail:1;unr:4,tail:1;stream:0;chunk:0;chunk:512" 2>&1 | grep "{"
timeout 600 python tools/spmm_bench.py --config C3 --p 4 --widths 44 --variants ";unr:4;tail:1;stream:0" 2>&1 | grep "{"
