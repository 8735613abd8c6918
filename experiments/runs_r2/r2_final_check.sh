#!/bin/bash
cd $GRAFT_REPO_ROOT 2>/dev/null || true
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/final_pytest.log 2>&1; tail -3 gpurun_out/final_pytest.log
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_final2.json 2> gpurun_out/bench_final2.err; echo bench rc=$?
python -c "
import json; d=json.load(open('gpurun_out/bench_final2.json')); c=d['coresident_p4']
print(d['value'], d['e2e']['value'], d['hoisted']['value'], d['roofline']['frac'], d['clocks'], c['value'], c['halo_kernels'])"
