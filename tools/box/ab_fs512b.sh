#!/bin/bash
# A/B/C at C3: default (8-column partner reads, PDL), + factorised signs at n=512, pre-PDL build d56999c
mkdir -p gpurun_out
for i in 1 2 3; do
  echo -n "d5:    " >> gpurun_out/ab_fs512b.txt; TSK_LIB=$PWD/ab/libtoesplit_d5.so timeout 300 python tools/launch_times.py c3 5 >> gpurun_out/ab_fs512b.txt 2>&1
  echo -n "base:  " >> gpurun_out/ab_fs512b.txt; timeout 300 python tools/launch_times.py c3 5 >> gpurun_out/ab_fs512b.txt 2>&1
  echo -n "fs512: " >> gpurun_out/ab_fs512b.txt; TSK_LIB=$PWD/ab/libtoesplit_fs512.so timeout 300 python tools/launch_times.py c3 5 >> gpurun_out/ab_fs512b.txt 2>&1
done
for lib in d5 base fs512; do
  L=$PWD/ab/libtoesplit_$lib.so; [ $lib = base ] && L=
  echo -n "$lib bench: " >> gpurun_out/ab_fs512b.txt
  TSK_LIB=$L timeout 300 python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --no-embed-baseline 2>/dev/null | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print(round(d['ms_per_step'],3), round(d['value'],2))" >> gpurun_out/ab_fs512b.txt
done
timeout 900 python -m pytest tests/test_split_gpu.py tests/test_fullsize_gpu.py -q -x -k "leaf or dyadic or partitions or fixture" > gpurun_out/ab_fs512b_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/ab_fs512b_pytest.log
