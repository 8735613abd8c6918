#!/bin/bash
cd $GRAFT_REPO_ROOT 2>/dev/null || true
timeout 900 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider -k "pipelined" 2>&1 | tail -2
for N in 2 4; do for K in 0 1 0 1; do
CDFGNN_INPUT_NCCL=$K timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port $((29700+RANDOM%200)) bench.py --gpus $N --steps 20 --warmup 5 --hoisted 0 > gpurun_out/ce_${N}_$K.json 2> gpurun_out/ce_${N}_$K.err
python -c "
import json
d=json.loads([l for l in open('gpurun_out/ce_${N}_$K.json') if l.startswith('{')][-1]); print('N=$N nccl_inputs=$K', d['value'], d['e2e']['value'])"
done; done
