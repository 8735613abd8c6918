#!/bin/bash
cd $GRAFT_REPO_ROOT 2>/dev/null || true
bash tools/scale.sh 4 20 cache_int8 > gpurun_out/r2_scale_final.log 2>&1
STEPS=10 bash tools/ablation.sh 4 C4:cache_int8 C4:nocache C5:cache_int8 C5:nocache > gpurun_out/r2_abl_final.log 2>&1
cat gpurun_out/r2_scale_final.log gpurun_out/r2_abl_final.log | cut -c1-400
