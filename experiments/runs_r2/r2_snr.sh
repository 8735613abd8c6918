#!/bin/bash
cd $GRAFT_REPO_ROOT 2>/dev/null || true
for snr in 0.005 0.01 0.02 0.05; do
  timeout 900 python tools/eps_study.py --config C3 --p 4 --epochs 60 --eps adaptive --snr $snr --out gpurun_out/snr_C3_$snr.json 2>&1 | grep '{' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('C3', d['snr'], d['final_acc'], d['acc_epochs'][::6], d['eps_epochs'][::6], d['avoided_frac_cache'])"
done
for snr in 0.05 0.1 0.2; do
  timeout 900 python tools/eps_study.py --config C4 --p 4 --epochs 60 --eps adaptive --snr $snr --out gpurun_out/snr_C4_$snr.json 2>&1 | grep '{' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('C4', d['snr'], d['final_acc'], d['acc_epochs'][::6], d['eps_epochs'][::6], d['avoided_frac_cache'])"
done
