#!/bin/bash
# ncu --set full of the 256-point leaf pass (C2, two CTAs per SM, 24 warps) for comparison
# with the 512-point one (12 warps)
mkdir -p gpurun_out
python tools/launch_times.py c2 1 > gpurun_out/ncu_leafc2_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_leaf1<float" -s 8 -c 1 -o /tmp/leafc2 python tools/launch_times.py c2 1 > gpurun_out/ncu_leafc2.log 2>&1
ncu -i /tmp/leafc2.ncu-rep --page raw --csv > gpurun_out/leafc2_raw.csv 2>&1
ncu -i /tmp/leafc2.ncu-rep --page source --csv --print-source sass > gpurun_out/leafc2_sass.csv 2>&1
gzip -f gpurun_out/leafc2_sass.csv
