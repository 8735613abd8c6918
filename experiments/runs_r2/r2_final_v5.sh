#!/bin/bash
# final 1-GPU validation of the round-2 code: smoke, pytest -m gpu, bench N=1
cd $GRAFT_REPO_ROOT 2>/dev/null || true
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_final_v5.log 2>&1; echo smoke rc=$?; tail -2 gpurun_out/smoke_final_v5.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_final_v5.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu_final_v5.log
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_final_v5.json 2> gpurun_out/bench_final_v5.err; echo bench rc=$?; cut -c1-400 gpurun_out/bench_final_v5.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_final_v5.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --hoisted 0 > gpurun_out/launches_final_v5.log 2>&1; echo ncu rc=$?
