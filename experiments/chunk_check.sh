#!/bin/bash
timeout 900 python tools/spmm_bench.py --config C3 --p 1 --widths 44,44 --variants "chunk:0;chunk:1024;chunk:4096;chunk:0" 2>&1 | grep "{"
timeout 600 python tools/spmm_bench.py --config C3 --p 2 --widths 44,256 --variants "chunk:0;chunk:512;chunk:2048;chunk:4096" 2>&1 | grep "{"
timeout 600 python tools/spmm_bench.py --config C3 --p 4 --widths 44,256 --variants "chunk:0;chunk:512;chunk:1024;chunk:2048" 2>&1 | grep "{"
timeout 600 python tools/spmm_bench.py --config C4 --p 4 --widths 48,256 --variants "chunk:0;chunk:512;chunk:2048" 2>&1 | grep "{"
