#!/bin/bash
# Evidence at HEAD: launch list of the bench command, ncu --set full of one whole C3 MVM
# (all ten launches: K1 x3, K2 x4, K3 x3), exported on the box; then the default bench line.
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-embed-baseline"
$CMD > gpurun_out/e_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/e_launches_bench_c3.csv $CMD > gpurun_out/e_ncu_launch.log 2>&1
echo "launch list rc=$?" >> gpurun_out/e_ncu_launch.log
python tools/launch_times.py c3 1 > gpurun_out/e_plain2.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_wtma|k_leaf1" -s 20 -c 10 -o /tmp/e_mvm python tools/launch_times.py c3 1 > gpurun_out/e_ncu_full.log 2>&1
echo "ncu full rc=$?" >> gpurun_out/e_ncu_full.log
ncu -i /tmp/e_mvm.ncu-rep --page raw --csv > gpurun_out/e_mvm_raw.csv 2>&1
ncu -i /tmp/e_mvm.ncu-rep --page source --csv --print-source sass > gpurun_out/e_mvm_sass.csv 2>&1
gzip -f gpurun_out/e_mvm_sass.csv
ls -la /tmp/e_mvm.ncu-rep >> gpurun_out/e_ncu_full.log
timeout 900 python bench.py > gpurun_out/e_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/e_bench.log
tail -c 600 gpurun_out/e_bench.log
