#!/bin/bash
# The other BASELINE configs with the round's final code: C2 (arxiv-shaped) at N = 1, 2;
# C4 (products-shaped) at N = 4 cache+int8 and no-cache; C5 at N = 4 cache+int8.
STEPS=10 bash tools/ablation.sh 1 C2:cache_int8 C2:nocache > gpurun_out/cf_c2_n1.log 2>&1
STEPS=10 bash tools/ablation.sh 2 C2:cache_int8 C2:nocache > gpurun_out/cf_c2_n2.log 2>&1
STEPS=5 bash tools/ablation.sh 4 C4:cache_int8 C4:nocache C5:cache_int8 > gpurun_out/cf_c45_n4.log 2>&1
