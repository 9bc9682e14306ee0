#!/bin/bash
# A/B at C2 (n = 256 TMA passes) + C3, tests of the TMA kernels
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_split_gpu.py -q -x -k "tma or wide_strided or wide_dyadic or partitions" > gpurun_out/ab_wtma2_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/ab_wtma2_pytest.log
for i in 1 2 3; do
  for c in c2 c3; do
  echo -n "$c wide: " >> gpurun_out/ab_wtma2.txt; TSK_NO_WTMA=1 timeout 300 python tools/launch_times.py $c 5 >> gpurun_out/ab_wtma2.txt 2>&1
  echo -n "$c wtma: " >> gpurun_out/ab_wtma2.txt; timeout 300 python tools/launch_times.py $c 5 >> gpurun_out/ab_wtma2.txt 2>&1
  done
done
timeout 900 python -m pytest tests/test_fullsize_gpu.py -q -x >> gpurun_out/ab_wtma2_pytest.log 2>&1
echo "fullsize rc=$?" >> gpurun_out/ab_wtma2_pytest.log
