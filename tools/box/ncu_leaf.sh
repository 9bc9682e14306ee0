#!/bin/bash
mkdir -p gpurun_out
python tools/launch_times.py c3 1 > gpurun_out/ncu_leaf_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_leaf1<float" -s 8 -c 1 -o gpurun_out/r02_leaf_xs python tools/launch_times.py c3 1 > gpurun_out/ncu_leaf.log 2>&1
echo rc=$? >> gpurun_out/ncu_leaf.log
