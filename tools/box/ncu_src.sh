#!/bin/bash
# ncu --set full with source of one C3 MVM's K1 (axis 1), K2 and K3 (axis 1)
mkdir -p gpurun_out
python tools/launch_times.py c3 1 > gpurun_out/ncu_src_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:k_wide<float|k_leaf1<float" -s 11 -c 4 -o gpurun_out/r02_src_c3 \
  python tools/launch_times.py c3 1 > gpurun_out/ncu_src.log 2>&1
echo rc=$? >> gpurun_out/ncu_src.log
