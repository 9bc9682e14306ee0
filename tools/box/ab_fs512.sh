#!/bin/bash
# A/B: leaf pass at n = 512 with factorised signs + 8-column partner reads (ab/libtoesplit_fs512.so) vs default
mkdir -p gpurun_out
for i in 1 2 3; do
  echo -n "base:  " >> gpurun_out/ab_fs512.txt; timeout 300 python tools/launch_times.py c3 5 >> gpurun_out/ab_fs512.txt 2>&1
  echo -n "fs512: " >> gpurun_out/ab_fs512.txt; TSK_LIB=$PWD/ab/libtoesplit_fs512.so timeout 300 python tools/launch_times.py c3 5 >> gpurun_out/ab_fs512.txt 2>&1
done
TSK_LIB=$PWD/ab/libtoesplit_fs512.so timeout 900 python -m pytest tests/test_split_gpu.py tests/test_fullsize_gpu.py -q -x -k "leaf or dyadic or partitions or fixture" > gpurun_out/ab_fs512_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/ab_fs512_pytest.log
