#!/bin/bash
# final 4-GPU validation: multi-GPU parity tests, C3 scaling N = 1/2/4, C4/C5 ablation at N = 4
cd $GRAFT_REPO_ROOT 2>/dev/null || true
timeout 2000 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider > gpurun_out/multi4_final_v5.log 2>&1; echo multi rc=$?; tail -2 gpurun_out/multi4_final_v5.log
bash tools/scale.sh 4 20 cache_int8 > gpurun_out/scale_final_v5.log 2>&1
STEPS=10 bash tools/ablation.sh 4 C4:cache_int8 C4:nocache C5:cache_int8 C5:nocache > gpurun_out/abl_final_v5.log 2>&1
cat gpurun_out/scale_final_v5.log gpurun_out/abl_final_v5.log | cut -c1-300
