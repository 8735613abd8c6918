#!/bin/bash
# Last check of the round on a 2-GPU box: full GPU suite, smoke, bench at N=1 and N=2.
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/fs_pytest.log 2>&1; echo rc=$? >> gpurun_out/fs_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fs_smoke.log 2>&1; echo rc=$? >> gpurun_out/fs_smoke.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/fs_bench_n1.json 2> gpurun_out/fs_bench_n1.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29690 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/fs_bench_n2.json 2> gpurun_out/fs_bench_n2.err
