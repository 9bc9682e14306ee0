#!/bin/bash
# A/B of the leaf sign variants + per-config bench lines + batch rates
mkdir -p gpurun_out
for i in 1 2; do
  for e in 0 1; do
    echo -n "NO_SF=$e: " >> gpurun_out/ab_sf2.txt
    TSK_LEAF_NO_SF=$e timeout 300 python tools/launch_times.py c3 5 >> gpurun_out/ab_sf2.txt 2>&1
  done
done
for c in c1 c2 c4 c3full; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-embed-baseline >> gpurun_out/r02_configs.jsonl 2> gpurun_out/r02_configs_$c.err
done
timeout 600 python tools/batch_rate.py c1 4 8 16 > gpurun_out/r02_batch.jsonl 2>&1
timeout 600 python tools/batch_rate.py c2 4 8 >> gpurun_out/r02_batch.jsonl 2>&1
timeout 900 python tools/batch_rate.py c3 2 4 8 >> gpurun_out/r02_batch.jsonl 2>&1
