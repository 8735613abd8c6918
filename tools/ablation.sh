#!/bin/bash
# Ablation / sweep runner: bench.py for each "CONFIG:MODE" at N GPUs (one JSON line each)
N=${1:-4}; shift
STEPS=${STEPS:-10}
for cm in "$@"; do
  C=${cm%%:*}; M=${cm##*:}
  OUT=gpurun_out/abl_${C}_${M}_n$N.json
  if [ $N -eq 1 ]; then
    timeout 1200 python bench.py --config $C --mode $M --steps $STEPS --warmup 3 --no-cpu-baseline --no-e2e > $OUT 2> ${OUT%.json}.err
  else
    timeout 1800 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port $((29700+RANDOM%200)) bench.py --gpus $N --config $C --mode $M --steps $STEPS --warmup 3 --no-e2e > $OUT 2> ${OUT%.json}.err
  fi
  echo "$C $M rc=$?"; python - "$OUT" <<'PY'
import json, sys
for l in open(sys.argv[1]):
    if l.startswith("{"):
        d = json.loads(l)
        print(json.dumps({k: d.get(k) for k in ["n_gpus", "value", "phase_ms", "comm_bytes_per_epoch",
                                                 "remote_accesses", "loss", "eps", "prep_s"]}))
PY
done
