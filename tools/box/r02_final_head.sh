#!/bin/bash
# Final HEAD check: smoke, full GPU suite, default bench line, reference arm
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/z_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/z_smoke.log
timeout 2400 python -m pytest tests -m gpu -q -rf --durations=10 > gpurun_out/z_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/z_pytest.log
timeout 900 python bench.py > gpurun_out/z_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/z_bench.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/z_bench_ref.log 2>&1
echo "ref rc=$?" >> gpurun_out/z_bench_ref.log
tail -3 gpurun_out/z_smoke.log; tail -4 gpurun_out/z_pytest.log; tail -c 400 gpurun_out/z_bench.log; tail -c 300 gpurun_out/z_bench_ref.log
