#!/bin/bash
cd $GRAFT_REPO_ROOT 2>/dev/null || true
for RL in none class; do
CMD="python tools/spmm_bench.py --config C4 --p 1 --relabel $RL --variants order:2 --widths 256 --reps 1"
$CMD > gpurun_out/c4loc_plain_$RL.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,l1tex__t_sector_hit_rate.pct,lts__throughput.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:spmm_kernel -c 2 --csv --log-file gpurun_out/c4loc_$RL.csv $CMD > /dev/null 2>&1; echo rc=$?
grep -v "^==" gpurun_out/c4loc_$RL.csv | cut -d, -f5,12-15 | tail -8
done
