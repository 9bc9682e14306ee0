#!/bin/bash
# full GPU suite, default bench, per-config lines, batch rates, launch times
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rf -s --durations=20 > gpurun_out/r02d_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02d_pytest.log
timeout 900 python bench.py > gpurun_out/r02d_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/r02d_bench.log
for c in c1 c2 c4 c3full; do
  timeout 600 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --no-embed-baseline >> gpurun_out/r02d_configs.jsonl 2> gpurun_out/r02d_configs_$c.err
done
timeout 600 python tools/batch_rate.py c1 4 8 16 > gpurun_out/r02d_batch.jsonl 2>&1
timeout 900 python tools/batch_rate.py c3 2 4 >> gpurun_out/r02d_batch.jsonl 2>&1
for c in c1 c2 c4 c3; do echo -n "$c " >> gpurun_out/r02d_launch_times.txt; timeout 300 python tools/launch_times.py $c 5 >> gpurun_out/r02d_launch_times.txt 2>&1; done
