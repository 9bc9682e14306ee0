#!/bin/bash
# pre-PDL build d56999c vs HEAD (PDL, factorised signs at 512, 8-column partner reads): C3 launches, bench lines c1/c4/c2/c3; full GPU suite
mkdir -p gpurun_out
for i in 1 2 3; do
  echo -n "d5:   " >> gpurun_out/ab_final.txt; TSK_LIB=$PWD/ab/libtoesplit_d5.so timeout 300 python tools/launch_times.py c3 5 >> gpurun_out/ab_final.txt 2>&1
  echo -n "head: " >> gpurun_out/ab_final.txt; timeout 300 python tools/launch_times.py c3 5 >> gpurun_out/ab_final.txt 2>&1
done
for i in 1 2; do
for c in c1 c4 c2 c3; do
  for lib in d5 head; do
    L=$PWD/ab/libtoesplit_$lib.so; [ $lib = head ] && L=
    echo -n "$c $lib bench: " >> gpurun_out/ab_final.txt
    TSK_LIB=$L timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --no-embed-baseline 2>/dev/null | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print(round(d['ms_per_step'],4), round(d['value'],2))" >> gpurun_out/ab_final.txt
  done
done
done
timeout 2400 python -m pytest tests -m gpu -q -x -rf > gpurun_out/ab_final_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/ab_final_pytest.log
