cd "$(dirname "$0")"
rm -f gpurun_out/search_ab.jsonl
timeout 300 python -m pytest tests/test_gpu_async.py tests/test_gpu_search.py -x -q > gpurun_out/r2_t8.log 2>&1
bash tests/search_ab.sh bida_search_fast_prev bida_search_fast_ts 3 > gpurun_out/search_ab.log 2>&1
bash tests/search_ab.sh bida_search_fast bida_search_fast_ts 3 >> gpurun_out/search_ab.log 2>&1
