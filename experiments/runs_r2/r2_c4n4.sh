#!/bin/bash
cd $GRAFT_REPO_ROOT 2>/dev/null || true
STEPS=10 bash tools/ablation.sh 4 C4:cache_int8 C3:cache_int8 > gpurun_out/r2_c4n4.log 2>&1
cat gpurun_out/r2_c4n4.log
