#!/bin/bash
# Scaling refresh on 4 GPUs: C3 at N=1,2,4 (cache+int8), C4 (products-shaped) at N=1,2,4,
# C5 ablation pair at N=4.
bash tools/scale.sh 4 10 cache_int8 > gpurun_out/r1h_scale.log 2>&1
for N in 1 2 4; do STEPS=5 bash tools/ablation.sh $N C4:cache_int8 >> gpurun_out/r1h_abl.log 2>&1; done
STEPS=5 bash tools/ablation.sh 4 C4:nocache C5:cache_int8 C5:nocache >> gpurun_out/r1h_abl.log 2>&1
