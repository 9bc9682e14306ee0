#!/bin/bash
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rf -s --durations=10 > gpurun_out/r02e_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02e_pytest.log
timeout 900 python bench.py > gpurun_out/r02e_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/r02e_bench.log
for c in c2 c3full; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-embed-baseline >> gpurun_out/r02e_configs.jsonl 2> gpurun_out/r02e_configs_$c.err
done
