#!/bin/bash
# Narrow-SpMM shape variants + ncu --set full of the halo kernels (co-resident C3 p=2, 1 GPU).
set -x
timeout 900 python tools/spmm_bench.py --config C3 --p 1 --widths 44 --variants ";shape:1;shape:2;shape:3" 2>&1 | grep "{" > gpurun_out/narrow_p1.jsonl
timeout 600 python tools/spmm_bench.py --config C3 --p 4 --widths 44 --variants ";shape:1;shape:2;shape:3" 2>&1 | grep "{" > gpurun_out/narrow_p4.jsonl
H2="python tools/halo_bench.py --config C3 --p 2 --epochs 2"
timeout 300 $H2 > gpurun_out/h2_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gather_pack|master_kernel|mirror_apply|scatter_pack" -s 8 -c 8 -o gpurun_out/halo_C3_p2 $H2 > gpurun_out/ncu_halo.log 2>&1
ls -la gpurun_out/
