#!/bin/bash
# MN-major ∇W: full GPU suite, smoke, bench C3 N=1 (and the K-major fallback), C4 N=1, C3 N=2.
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/mn_pytest.log 2>&1; echo rc=$? >> gpurun_out/mn_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/mn_smoke.log 2>&1; echo rc=$? >> gpurun_out/mn_smoke.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/mn_bench_n1.json 2> gpurun_out/mn_bench_n1.err
CDFGNN_WGRAD_KMAJOR=1 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --hoisted 0 --no-e2e > gpurun_out/mn_bench_n1_kmajor.json 2> gpurun_out/mn_bench_n1_kmajor.err
timeout 900 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline --hoisted 0 --no-e2e > gpurun_out/mn_bench_c4.json 2> gpurun_out/mn_bench_c4.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29695 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/mn_bench_n2.json 2> gpurun_out/mn_bench_n2.err
