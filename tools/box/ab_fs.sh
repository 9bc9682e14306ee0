#!/bin/bash
# A/B: leaf pass with factorised signs (default) vs per-value flips (TSK_LEAF_NO_FS=1)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_split_gpu.py -q -x -k "leaf or dyadic or partitions" > gpurun_out/ab_fs_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/ab_fs_pytest.log
for i in 1 2 3; do
  for c in c3 c2; do
  echo -n "$c nofs: " >> gpurun_out/ab_fs.txt; TSK_LEAF_NO_FS=1 timeout 300 python tools/launch_times.py $c 5 >> gpurun_out/ab_fs.txt 2>&1
  echo -n "$c fs:   " >> gpurun_out/ab_fs.txt; timeout 300 python tools/launch_times.py $c 5 >> gpurun_out/ab_fs.txt 2>&1
  done
done
timeout 900 python -m pytest tests/test_fullsize_gpu.py -q -x -k fixture >> gpurun_out/ab_fs_pytest.log 2>&1
echo "fullsize rc=$?" >> gpurun_out/ab_fs_pytest.log
