#!/bin/bash
# A/B: FMA-fused radix-8 tail (e +- h t as FFMA2) and fused odd-branch emit (e + conj(P) o
# with e on the first FFMA2) — HEAD build vs the previous build (ab/libtoesplit_head.so)
mkdir -p gpurun_out
out=gpurun_out/ab_fuse.txt
for cfg in c3 c2 c1 c4; do
  echo "== $cfg" >> $out
  for i in 1 2 3; do
    echo -n "head: " >> $out; TSK_LIB=$PWD/ab/libtoesplit_head.so timeout 300 python tools/launch_times.py $cfg 5 2>&1 | tail -n 1 >> $out
    echo -n "fuse: " >> $out; timeout 300 python tools/launch_times.py $cfg 5 2>&1 | tail -n 1 >> $out
  done
done
timeout 1200 python -m pytest tests/test_split_gpu.py tests/test_engine_gpu.py tests/test_fullsize_gpu.py -q -x > gpurun_out/ab_fuse_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/ab_fuse_pytest.log
