#!/bin/bash
cd $GRAFT_REPO_ROOT 2>/dev/null || true
timeout 1500 python tools/eps_study.py --config C4 --p 4 --epochs 60 --eps adaptive,0,0.001,0.01,0.03,0.1,0.3 --quant 8 --snr 0.05 --out gpurun_out/eps_study_C4_p4_snr0.05_B8.json 2>&1 | grep '{' | cut -c1-400
timeout 1500 python tools/eps_study.py --config C4 --p 4 --epochs 60 --eps adaptive,0.03 --quant 4,16,0 --snr 0.05 --out gpurun_out/eps_study_C4_p4_snr0.05_Bvar.json 2>&1 | grep '{' | cut -c1-400
timeout 1500 python tools/eps_study.py --config C3 --p 4 --epochs 60 --eps adaptive,0,0.01,0.1,0.3 --quant 8 --snr 0.005 --out gpurun_out/eps_study_C3_p4_snr0.005_B8.json 2>&1 | grep '{' | cut -c1-400
