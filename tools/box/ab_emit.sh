#!/bin/bash
# A/B: d = 3 closed-form orbit geometry in the 512-point FS leaf (HEAD build) vs previous build
mkdir -p gpurun_out
for i in 1 2 3; do
  echo -n "prev: " >> gpurun_out/ab_emit.txt; TSK_LIB=$PWD/ab/libtoesplit_prev.so timeout 300 python tools/launch_times.py c3 5 >> gpurun_out/ab_emit.txt 2>&1
  echo -n "emit: " >> gpurun_out/ab_emit.txt; timeout 300 python tools/launch_times.py c3 5 >> gpurun_out/ab_emit.txt 2>&1
done
timeout 900 python -m pytest tests/test_split_gpu.py tests/test_engine_gpu.py tests/test_fullsize_gpu.py -q -x -k "leaf or dyadic or batch or fixture or partitions" > gpurun_out/ab_emit_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/ab_emit_pytest.log
