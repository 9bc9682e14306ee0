#!/bin/bash
# Final round-2 measurements: default bench (30 steps), per-config lines, batch rates,
# launch list of the bench command, ncu full capture of K3 (k_wtma<512,1>) exported on the box
mkdir -p gpurun_out
timeout 900 python bench.py --steps 30 --warmup 5 > gpurun_out/f_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/f_bench.log
timeout 600 python bench.py > gpurun_out/f_bench_default.log 2>&1
for c in c1 c1m c2 c4 c3full; do
  timeout 600 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --no-embed-baseline >> gpurun_out/f_configs.jsonl 2> gpurun_out/f_configs_$c.err
done
for c in c1 c2 c4 c3; do timeout 300 python tools/launch_times.py $c 5 >> gpurun_out/f_launch_times.txt 2>&1; done
timeout 600 python tools/batch_rate.py c1 4 8 16 > gpurun_out/f_batch.jsonl 2>&1
timeout 900 python tools/batch_rate.py c3 2 4 8 >> gpurun_out/f_batch.jsonl 2>&1
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-embed-baseline"
$CMD > gpurun_out/f_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/f_launches_bench_c3.csv $CMD > gpurun_out/f_ncu_launch.log 2>&1
python tools/launch_times.py c3 1 > gpurun_out/f_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_wtma<.int.512, .int.1>" -s 2 -c 1 -o /tmp/f_k3 python tools/launch_times.py c3 1 > gpurun_out/f_ncu_k3.log 2>&1
ncu -i /tmp/f_k3.ncu-rep --page raw --csv > gpurun_out/f_k3_raw.csv 2>&1
ncu -i /tmp/f_k3.ncu-rep --page source --csv --print-source sass > gpurun_out/f_k3_sass.csv 2>&1
gzip -f gpurun_out/f_k3_sass.csv
echo done >> gpurun_out/f_ncu_k3.log
