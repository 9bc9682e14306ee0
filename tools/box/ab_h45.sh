#!/bin/bash
# A/B on one box: previous build (head), fused emit (fuse), + 45-degree twiddle factors on the
# next butterfly (tree build), + streaming output stores (stcs)
mkdir -p gpurun_out
out=gpurun_out/ab_h45.txt
for cfg in c3 c2; do
  echo "== $cfg" >> $out
  for i in 1 2 3; do
    for v in head fuse stcs; do
      echo -n "$v: " >> $out; TSK_LIB=$PWD/ab/libtoesplit_$v.so timeout 300 python tools/launch_times.py $cfg 5 2>&1 | tail -n 1 >> $out
    done
    echo -n "h45:  " >> $out; timeout 300 python tools/launch_times.py $cfg 5 2>&1 | tail -n 1 >> $out
  done
done
timeout 1200 python -m pytest tests/test_split_gpu.py tests/test_engine_gpu.py tests/test_fullsize_gpu.py -q -x > gpurun_out/ab_h45_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/ab_h45_pytest.log
