#!/bin/bash
cd $GRAFT_REPO_ROOT 2>/dev/null || true
for C in C3 C4; do for O in "" "--overlap"; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port $((29800+RANDOM%100)) bench.py --gpus 4 --config $C --steps 10 --warmup 3 --no-e2e --hoisted 0 $O > gpurun_out/ovl_${C}${O}.json 2> gpurun_out/ovl_${C}${O}.err
python -c "
import json,sys
d=json.loads([l for l in open('gpurun_out/ovl_${C}${O}.json') if l.startswith('{')][-1]); print('$C', '$O', d['value'], d['phase_ms'], d['config']['overlap'])"
done; done
