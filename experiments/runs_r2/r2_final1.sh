#!/bin/bash
cd $GRAFT_REPO_ROOT 2>/dev/null || true
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_r2.log 2>&1; echo smoke rc=$?; tail -2 gpurun_out/smoke_r2.log
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo bench rc=$?
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/ref_final.json 2> gpurun_out/ref_final.err; echo ref rc=$?
cat gpurun_out/ref_final.json | cut -c1-600
