#!/bin/bash
# HEAD check: full GPU suite, default bench line, launch list of the bench command
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rf --durations=15 > gpurun_out/r02h_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02h_pytest.log
timeout 900 python bench.py > gpurun_out/r02h_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/r02h_bench.log
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-embed-baseline"
$CMD > gpurun_out/r02h_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02h_launches_bench_c3.csv $CMD > gpurun_out/r02h_ncu_launch.log 2>&1
echo "ncu rc=$?" >> gpurun_out/r02h_ncu_launch.log
