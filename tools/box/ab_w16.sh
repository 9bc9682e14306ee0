#!/bin/bash
# A/B: TMA strided passes with 16-column tiles (128 B rows, 256 threads, two CTAs per SM)
# against the 32-column default (256 B rows, one CTA per SM)
mkdir -p gpurun_out
out=gpurun_out/ab_w16.txt
TSK_LIB=$PWD/ab/libtoesplit_w16.so timeout 300 python tools/family_cases.py wtma > gpurun_out/ab_w16_cases.txt 2>&1
for cfg in c3 c2; do
  echo "== $cfg" >> $out
  for i in 1 2 3; do
    for v in tree w16; do
      echo -n "$v: " >> $out; TSK_LIB=$PWD/ab/libtoesplit_$v.so timeout 300 python tools/launch_times.py $cfg 5 2>&1 | tail -n 1 >> $out
    done
  done
done
