#!/bin/bash
# A/B: the leaf pass's x-row prefetch issued by the component-2 warps (xc2) instead of the
# component-0 warps (tree)
mkdir -p gpurun_out
out=gpurun_out/ab_xc.txt
for cfg in c3 c2; do
  echo "== $cfg" >> $out
  for i in 1 2 3 4; do
    for v in tree xc2; do
      echo -n "$v: " >> $out; TSK_LIB=$PWD/ab/libtoesplit_$v.so timeout 300 python tools/launch_times.py $cfg 5 2>&1 | tail -n 1 >> $out
    done
  done
done
TSK_LIB=$PWD/ab/libtoesplit_xc2.so timeout 300 python tools/family_cases.py > gpurun_out/ab_xc_cases.txt 2>&1
