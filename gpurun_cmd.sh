#!/bin/bash
cd "$(dirname "$0")"
mkdir -p gpurun_out
rm -f gpurun_out/search_ab.jsonl
bash tests/search_ab.sh bida_search_fast_old bida_search_fast 3 > gpurun_out/search_ab.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_search.py tests/test_gpu_search_configs.py -q -x > gpurun_out/search_tests.log 2>&1
