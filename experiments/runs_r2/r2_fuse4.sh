#!/bin/bash
cd $GRAFT_REPO_ROOT 2>/dev/null || true
for C in C3 C4; do for F in 1 0 1 0; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port $((29900+RANDOM%90)) bench.py --gpus 4 --config $C --steps 20 --warmup 5 --no-e2e --hoisted 0 --fuse $F > gpurun_out/f4_${C}_$F.json 2> gpurun_out/f4_${C}_$F.err
python -c "
import json
d=json.loads([l for l in open('gpurun_out/f4_${C}_$F.json') if l.startswith('{')][-1]); print('$C fuse=$F', d['value'], d['phase_ms']['spmm'], d['phase_ms']['sync'])"
done; done
