#!/bin/bash
# Round 2: scaling N=1,2,4 (C3, cache_int8) + C4 N=4 cache/no-cache + C5 N=4 ablation
cd $GRAFT_REPO_ROOT 2>/dev/null || true
bash tools/scale.sh 4 10 cache_int8 > gpurun_out/r2_scale.log 2>&1
STEPS=10 bash tools/ablation.sh 4 C4:cache_int8 C4:nocache C5:cache_int8 C5:nocache C5:quant_only C5:cache_fp32 > gpurun_out/r2_abl4.log 2>&1
tail -50 gpurun_out/r2_scale.log gpurun_out/r2_abl4.log
