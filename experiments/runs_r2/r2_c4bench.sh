#!/bin/bash
cd $GRAFT_REPO_ROOT 2>/dev/null || true
python bench.py --config C4 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --hoisted 0 > gpurun_out/bench_C4_n1.json 2> gpurun_out/bench_C4_n1.err; echo rc=$?
python -c "
import json; d=json.load(open('gpurun_out/bench_C4_n1.json')); c=d['coresident_p4']
print(d['value'], d['phase_ms']); print(json.dumps(c['halo_kernels'])); print(c['value'], c['phase_ms'])"
