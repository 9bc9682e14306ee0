#!/bin/bash
# GPU suite, default bench, launch list and one ncu --set full capture of one C3 MVM
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rf -s --durations=20 > gpurun_out/r02b_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02b_pytest.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r02b_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/r02b_bench.log
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-embed-baseline"
$CMD > gpurun_out/r02b_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches_bench_c3.csv $CMD > gpurun_out/r02b_ncu_launch.log 2>&1
python tools/launch_times.py c3 1 > gpurun_out/r02b_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_wide<float|k_leaf1<float" -s 20 -c 10 -o gpurun_out/r02_full_c3 python tools/launch_times.py c3 1 > gpurun_out/r02b_ncu_full.log 2>&1
echo done >> gpurun_out/r02b_ncu_full.log
