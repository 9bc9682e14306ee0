#!/bin/bash
# Run on the GPU box (gpurun): the C3 (512^3) reference fixture needs ~80 GB of
# host RAM. Refuses to start below 160 GB available and caps the address space
# so a shortfall ends in bad_alloc, not the OOM killer.
mkdir -p gpurun_out
{
  nproc; free -g; lscpu | grep -E "Model name|Socket|Thread|Core"; nvidia-smi --query-gpu=name,memory.total --format=csv
} > gpurun_out/box_info.txt 2>&1
avail=$(awk '/MemAvailable/ {print int($2/1048576)}' /proc/meminfo)
echo "MemAvailable ${avail} GB" >> gpurun_out/box_info.txt
if [ "$avail" -lt 160 ]; then echo "not enough host RAM for c3" >> gpurun_out/box_info.txt; exit 3; fi
ulimit -v $((140 * 1024 * 1024))
python tests/golden/make_fullsize.py c3 --out gpurun_out/c3_512x512x512_ref.npz > gpurun_out/c3_fixture.log 2>&1
echo "rc=$?" >> gpurun_out/c3_fixture.log
