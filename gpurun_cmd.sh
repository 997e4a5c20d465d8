cd "$(dirname "$0")"
timeout 600 python -m pytest tests/test_gpu_walks.py tests/test_gpu_linear.py tests/test_gpu_search_configs.py -x -q > gpurun_out/r2_t3.log 2>&1
timeout 900 python bench.py > gpurun_out/r2_bench3.json 2> gpurun_out/r2_bench3.err
python tests/small_batch_launches.py > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_small_launches.csv python tests/small_batch_launches.py > gpurun_out/ncu_small.log 2>&1
