#!/bin/bash
# Scaling sweep: bench.py at N = 1..max GPUs of this box (one JSON line per N).
MAXG=${1:-8}
STEPS=${2:-10}
MODE=${3:-cache_int8}
for N in 1 2 4 8; do
  if [ $N -gt $MAXG ]; then break; fi
  if [ $N -eq 1 ]; then
    timeout 600 python bench.py --steps $STEPS --warmup 3 --no-cpu-baseline --mode $MODE > gpurun_out/scale_${MODE}_n$N.json 2> gpurun_out/scale_${MODE}_n$N.err
  else
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port $((29600+N)) bench.py --gpus $N --steps $STEPS --warmup 3 --mode $MODE > gpurun_out/scale_${MODE}_n$N.json 2> gpurun_out/scale_${MODE}_n$N.err
  fi
  echo "N=$N rc=$?"; cat gpurun_out/scale_${MODE}_n$N.json | python -c "import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(json.dumps({k:d.get(k) for k in ['n_gpus','value','phase_ms','comm_bytes_per_epoch','remote_accesses','nvlink','e2e']}))"
done
