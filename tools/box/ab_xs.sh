#!/bin/bash
mkdir -p gpurun_out
for i in 1 2 3; do
  echo -n "base: " >> gpurun_out/ab_xs.txt; timeout 300 python tools/launch_times.py c3 5 >> gpurun_out/ab_xs.txt 2>&1
  echo -n "xs:   " >> gpurun_out/ab_xs.txt; TSK_LIB=$PWD/ab/libtoesplit_xs.so timeout 300 python tools/launch_times.py c3 5 >> gpurun_out/ab_xs.txt 2>&1
done
TSK_LIB=$PWD/ab/libtoesplit_xs.so timeout 1200 python -m pytest tests/test_fullsize_gpu.py tests/test_split_gpu.py tests/test_engine_gpu.py -q -x -k "c3 or fixture or leaf or dyadic or batch or partition or fuzz" > gpurun_out/ab_xs_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/ab_xs_pytest.log
