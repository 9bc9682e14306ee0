#!/bin/bash
# A/B timing of library builds on one box: tools/ab.sh libA.so libB.so [reps]
# Prints per-family ms for each run (alternating A, B).
reps=${3:-2}
for i in $(seq 1 $reps); do
  for lib in "$1" "$2"; do
    TSK_LIB=$PWD/$lib timeout 200 python bench.py --steps 5 --warmup 3 2>/dev/null | python -c "
import json,sys
d=json.loads([l for l in sys.stdin if l.startswith('{')][-1])
f=d['kernel_families']
print('$lib', round(d['ms_per_step'],2), ' '.join(f'{k}={v[\"ms\"]:.2f}' for k,v in f.items()))"
  done
done
