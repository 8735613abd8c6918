#!/bin/bash
# N=2 bench with and without the boundary-rows-first overlap, plus co-resident halo timing.
for o in "" "--no-overlap"; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 2 --steps 10 --warmup 3 --no-e2e $o > gpurun_out/ovl$o.json 2> gpurun_out/ovl$o.err
  python -c "
import json
for l in open('gpurun_out/ovl$o.json'):
    if l.startswith('{'):
        d=json.loads(l); print('$o', d['value'], json.dumps(d['phase_ms']))"
done
for o in 1 0; do timeout 300 python tools/halo_bench.py --config C3 --p 2 --epochs 3 --overlap $o | tail -1; done
