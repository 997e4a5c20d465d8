cd "$(dirname "$0")"
rm -f gpurun_out/async_sweep.jsonl gpurun_out/search_configs.jsonl
timeout 900 python -m pytest tests/test_gpu_search.py tests/test_gpu_search_configs.py tests/test_gpu_async.py -x -q > gpurun_out/r2_t5.log 2>&1
bash tests/search_async_sweep.sh > gpurun_out/async_sweep.log 2>&1
