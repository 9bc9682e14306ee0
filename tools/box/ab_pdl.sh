#!/bin/bash
# A/B: programmatic dependent launch (default) vs plain launches (TSK_NO_PDL=1); full GPU suite
mkdir -p gpurun_out
for i in 1 2 3; do
  for c in c1 c4 c2 c3; do
    echo -n "$c nopdl: " >> gpurun_out/ab_pdl2.txt; TSK_NO_PDL=1 timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --no-embed-baseline 2>/dev/null | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print(round(d['ms_per_step'],4), round(d['value'],1))" >> gpurun_out/ab_pdl2.txt
    echo -n "$c pdl:   " >> gpurun_out/ab_pdl2.txt; timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --no-embed-baseline 2>/dev/null | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print(round(d['ms_per_step'],4), round(d['value'],1))" >> gpurun_out/ab_pdl2.txt
  done
done
timeout 1200 python -m pytest tests/test_engine_gpu.py tests/test_split_gpu.py tests/test_capi_ref_gpu.py -q -x -rf > gpurun_out/ab_pdl2_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/ab_pdl2_pytest.log
