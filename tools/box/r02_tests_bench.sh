#!/bin/bash
# GPU suite + default bench on the box; logs into gpurun_out/
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rf --durations=15 > gpurun_out/r02_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02_pytest.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r02_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/r02_bench.log
