#!/bin/bash
# A/B: TMA-landing strided passes (default) vs k_wide (TSK_NO_WTMA=1); tests
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_split_gpu.py -q -x -k "tma or wide_strided or wide_dyadic or partitions" > gpurun_out/ab_wtma_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/ab_wtma_pytest.log
for i in 1 2 3; do
  echo -n "wide: " >> gpurun_out/ab_wtma.txt; TSK_NO_WTMA=1 timeout 300 python tools/launch_times.py c3 5 >> gpurun_out/ab_wtma.txt 2>&1
  echo -n "wtma: " >> gpurun_out/ab_wtma.txt; timeout 300 python tools/launch_times.py c3 5 >> gpurun_out/ab_wtma.txt 2>&1
done
timeout 600 python -m pytest tests/test_fullsize_gpu.py -q -x -k "fixture" >> gpurun_out/ab_wtma_pytest.log 2>&1
echo "fullsize rc=$?" >> gpurun_out/ab_wtma_pytest.log
