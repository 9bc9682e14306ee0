#!/bin/bash
mkdir -p gpurun_out
for i in 1 2 3; do
  for e in 0 1; do
    echo -n "NO_SF=$e: " >> gpurun_out/ab_sf.txt
    TSK_LEAF_NO_SF=$e timeout 300 python tools/launch_times.py c3 5 >> gpurun_out/ab_sf.txt 2>&1
  done
done
timeout 300 python tools/launch_times.py c2 5 >> gpurun_out/ab_sf.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x -rf -s -k "fullsize_vs_reference or dyadic or leaf or compressed or partition or fuzz or engine or tskf or capi" > gpurun_out/r02_pytest_sf.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02_pytest_sf.log
