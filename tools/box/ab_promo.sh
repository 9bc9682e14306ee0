#!/bin/bash
# A/B of the TMA tile loads of the strided passes: L2 promotion none / 128 B / 256 B (tree),
# 64-row boxes (box64) instead of 256-row ones
mkdir -p gpurun_out
out=gpurun_out/ab_promo.txt
for cfg in c3 c2; do
  echo "== $cfg" >> $out
  for i in 1 2 3; do
    for v in tree promo0 promo2 box64; do
      echo -n "$v: " >> $out; TSK_LIB=$PWD/ab/libtoesplit_$v.so timeout 300 python tools/launch_times.py $cfg 5 2>&1 | tail -n 1 >> $out
    done
  done
done
