#!/bin/bash
mkdir -p gpurun_out
for c in c1 c1m; do
CMD="python tools/launch_times.py $c 3"
$CMD > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k "regex:k_wide|k_leaf1|k_wtma|k_fast|k_strided" --csv --log-file gpurun_out/${c}_ncu_list.csv $CMD > /dev/null 2>&1
done
echo done
