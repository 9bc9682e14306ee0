#!/bin/bash
# A/B: leaf split barrier (mbarrier-completed spectra staging + fiber-pair barrier; default) vs unit barrier
mkdir -p gpurun_out
for i in 1 2 3; do for c in c3 c2; do
  echo -n "$c nosb: " >> gpurun_out/ab_sb.txt; TSK_LIB=$PWD/ab/libtoesplit_nosb.so timeout 300 python tools/launch_times.py $c 5 >> gpurun_out/ab_sb.txt 2>&1
  echo -n "$c sb:   " >> gpurun_out/ab_sb.txt; timeout 300 python tools/launch_times.py $c 5 >> gpurun_out/ab_sb.txt 2>&1
done; done
timeout 900 python -m pytest tests/test_split_gpu.py tests/test_fullsize_gpu.py tests/test_engine_gpu.py -q -x -k "leaf or dyadic or partitions or fixture or batch" > gpurun_out/ab_sb_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/ab_sb_pytest.log
