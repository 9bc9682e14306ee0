#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_embed_gpu.py tests/test_split_gpu.py tests/test_engine_gpu.py tests/test_acceptance_gpu.py -q -x -rf > gpurun_out/r02c_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02c_pytest.log
timeout 600 python tools/embed_compare.py c1 20 > gpurun_out/r02_embed_compare.jsonl 2>&1
timeout 900 python tools/embed_compare.py c3 3 >> gpurun_out/r02_embed_compare.jsonl 2>&1
