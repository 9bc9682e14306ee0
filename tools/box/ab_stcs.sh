#!/bin/bash
# A/B on one box: previous build (head, plain stores), tree build (streaming stores in K1 and the
# N >= 256 leaf), stcs3 (also in K3), ldef (tree + L2 evict-first policy on the TMA / bulk loads)
mkdir -p gpurun_out
out=gpurun_out/ab_stcs.txt
for cfg in c3 c2; do
  echo "== $cfg" >> $out
  for i in 1 2 3; do
    for v in head stcs3 ldef; do
      echo -n "$v: " >> $out; TSK_LIB=$PWD/ab/libtoesplit_$v.so timeout 300 python tools/launch_times.py $cfg 5 2>&1 | tail -n 1 >> $out
    done
    echo -n "tree: " >> $out; timeout 300 python tools/launch_times.py $cfg 5 2>&1 | tail -n 1 >> $out
  done
done
# ncu source-level capture of the tree build's leaf pass
python tools/launch_times.py c3 1 > gpurun_out/ncu_leaf3_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_leaf1<float" -s 8 -c 1 -o /tmp/leaf3 python tools/launch_times.py c3 1 > gpurun_out/ncu_leaf3.log 2>&1
ncu -i /tmp/leaf3.ncu-rep --page raw --csv > gpurun_out/leaf3_raw.csv 2>&1
ncu -i /tmp/leaf3.ncu-rep --page source --csv --print-source sass > gpurun_out/leaf3_sass.csv 2>&1
gzip -f gpurun_out/leaf3_sass.csv
