#!/bin/bash
cd $GRAFT_REPO_ROOT 2>/dev/null || true
for K in 0 1; do
CDFGNN_INPUT_PCIE_ONLY=$K timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port $((29850+K)) bench.py --gpus 4 --steps 10 --warmup 3 --hoisted 0 > gpurun_out/e2e4_$K.json 2> gpurun_out/e2e4_$K.err
python -c "
import json
d=json.loads([l for l in open('gpurun_out/e2e4_$K.json') if l.startswith('{')][-1]); print('pcie_only=$K', d['value'], d['e2e']['value'], d['e2e']['serial_value'], d['e2e']['h2d_bytes_per_step'])"
done
