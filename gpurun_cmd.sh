#!/bin/bash
cd "$(dirname "$0")"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_search.py tests/test_gpu_search_configs.py -q -x > gpurun_out/search_tests.log 2>&1
