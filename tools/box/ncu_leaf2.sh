#!/bin/bash
mkdir -p gpurun_out
python tools/launch_times.py c3 1 > gpurun_out/ncu_leaf2_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_leaf1<float" -s 8 -c 1 -o /tmp/leaf2 python tools/launch_times.py c3 1 > gpurun_out/ncu_leaf2.log 2>&1
ncu -i /tmp/leaf2.ncu-rep --page raw --csv > gpurun_out/leaf2_raw.csv 2>&1
ncu -i /tmp/leaf2.ncu-rep --page source --csv --print-source sass > gpurun_out/leaf2_sass.csv 2>&1
gzip -f gpurun_out/leaf2_sass.csv
