#!/bin/bash
mkdir -p gpurun_out
python tools/embed_compare.py c3 3 > gpurun_out/embed_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled \
  -k "regex:k_contig|k_wide<float, 1024|k_block_symbol|k_embed_corner" -c 40 --csv \
  --log-file gpurun_out/r02_embed_launches.csv python tools/embed_compare.py c3 3 > gpurun_out/embed_ncu.log 2>&1
