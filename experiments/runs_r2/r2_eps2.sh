#!/bin/bash
cd $GRAFT_REPO_ROOT 2>/dev/null || true
timeout 1500 python tools/eps_study.py --config C4 --p 4 --epochs 60 --eps adaptive,0 --quant 8 --snr 0.05 --out gpurun_out/eps_dbg.json > gpurun_out/eps_dbg.log 2>&1; echo rc=$?; tail -30 gpurun_out/eps_dbg.log | cut -c1-300
