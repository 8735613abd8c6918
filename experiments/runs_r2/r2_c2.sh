#!/bin/bash
# C2 (ogbn-arxiv-shaped) at N = 1 and 2, cache + int8 and no cache, final code
cd $GRAFT_REPO_ROOT 2>/dev/null || true
STEPS=20 bash tools/ablation.sh 1 C2:cache_int8 C2:nocache > gpurun_out/c2_n1.log 2>&1
STEPS=20 bash tools/ablation.sh 2 C2:cache_int8 C2:nocache > gpurun_out/c2_n2.log 2>&1
cat gpurun_out/c2_n1.log gpurun_out/c2_n2.log | cut -c1-300
