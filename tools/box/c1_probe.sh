#!/bin/bash
mkdir -p gpurun_out
for c in c1 c1m c1 c1m; do timeout 300 python bench.py --config $c --steps 200 --warmup 20 --no-e2e --no-cpu-baseline --no-embed-baseline 2>/dev/null | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print('$c', round(d['ms_per_step'],4), round(d['value'],1), d['step_roofline']['frac'])" >> gpurun_out/c1_probe.txt; done
python tools/launch_times.py c1 20 >> gpurun_out/c1_probe.txt 2>&1
python tools/launch_times.py c1m 20 >> gpurun_out/c1_probe.txt 2>&1
CMD="python bench.py --config c1 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-embed-baseline"
$CMD > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size --clock-control none -c 200 --csv --log-file gpurun_out/c1_launches.csv $CMD > /dev/null 2>&1
echo done >> gpurun_out/c1_probe.txt
