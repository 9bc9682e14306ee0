#!/bin/bash
# default bench line, per-config lines, launch list, ncu full capture of one C3 MVM's passes
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/m2_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/m2_bench.log
for c in c1 c2 c4 c3full; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-embed-baseline >> gpurun_out/m2_configs.jsonl 2> gpurun_out/m2_configs_$c.err
done
for c in c1 c2 c4 c3; do timeout 300 python tools/launch_times.py $c 5 >> gpurun_out/m2_launch_times.txt 2>&1; done
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-embed-baseline"
$CMD > gpurun_out/m2_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/m2_launches_bench_c3.csv $CMD > gpurun_out/m2_ncu_launch.log 2>&1
python tools/launch_times.py c3 1 > gpurun_out/m2_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_wtma|k_leaf1<float" -s 10 -c 4 -o /tmp/r02_full_c3_wtma python tools/launch_times.py c3 1 > gpurun_out/m2_ncu_full.log 2>&1
echo "done rc=$?" >> gpurun_out/m2_ncu_full.log
ncu -i /tmp/r02_full_c3_wtma.ncu-rep --page raw --csv > gpurun_out/m2_ncu_full_raw.csv 2>&1
ncu -i /tmp/r02_full_c3_wtma.ncu-rep --page source --csv --print-source sass > gpurun_out/m2_ncu_full_sass.csv 2>&1
gzip -f gpurun_out/m2_ncu_full_sass.csv
