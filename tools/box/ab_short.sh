#!/bin/bash
mkdir -p gpurun_out
for i in 1 2 3; do for c in c1 c1m; do for lib in noshort head; do
  L=$PWD/ab/libtoesplit_$lib.so; [ $lib = head ] && L=
  echo -n "$c $lib: " >> gpurun_out/ab_short.txt
  TSK_LIB=$L TSK_DEBUG_OCC=1 timeout 300 python bench.py --config $c --steps 200 --warmup 20 --no-e2e --no-cpu-baseline --no-embed-baseline 2>gpurun_out/ab_short_$lib.err | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print(round(d['ms_per_step'],4), round(d['value'],1))" >> gpurun_out/ab_short.txt
done; done; done
timeout 900 python -m pytest tests/test_split_gpu.py tests/test_engine_gpu.py -q -x -k "leaf or dyadic or c1 or batch or graph" > gpurun_out/ab_short_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/ab_short_pytest.log
