#!/bin/bash
# A/B: x-prefetch geometry on component-0 warps only (HEAD build) vs previous build; c3full with/without PDL
mkdir -p gpurun_out
for i in 1 2 3; do
  echo -n "prev: " >> gpurun_out/ab_ix.txt; TSK_LIB=$PWD/ab/libtoesplit_prev.so timeout 300 python tools/launch_times.py c3 5 >> gpurun_out/ab_ix.txt 2>&1
  echo -n "ix:   " >> gpurun_out/ab_ix.txt; timeout 300 python tools/launch_times.py c3 5 >> gpurun_out/ab_ix.txt 2>&1
done
for i in 1 2; do for lib in prev ix; do
  L=$PWD/ab/libtoesplit_$lib.so; [ $lib = ix ] && L=
  echo -n "c3 $lib bench: " >> gpurun_out/ab_ix.txt
  TSK_LIB=$L timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-embed-baseline 2>/dev/null | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print(round(d['ms_per_step'],3), round(d['value'],2), d['clocks']['reasons'])" >> gpurun_out/ab_ix.txt
done; done
for pdl in 0 1; do
  echo -n "c3full nopdl=$pdl: " >> gpurun_out/ab_ix.txt
  TSK_NO_PDL=$pdl timeout 600 python bench.py --config c3full --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-embed-baseline 2>/dev/null | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print(round(d['ms_per_step'],3), round(d['value'],2), d['clocks'], round(sum(v['ms'] for v in d['kernel_families'].values()),2))" >> gpurun_out/ab_ix.txt
done
timeout 900 python -m pytest tests/test_split_gpu.py tests/test_engine_gpu.py -q -x -k "leaf or dyadic or batch" > gpurun_out/ab_ix_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/ab_ix_pytest.log
