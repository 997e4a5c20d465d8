cd "$(dirname "$0")"
rm -f gpurun_out/host_sweep.jsonl gpurun_out/search_configs.jsonl
timeout 600 python -m pytest tests/test_gpu_async.py tests/test_gpu_linear.py tests/test_gpu_pdb.py "tests/test_gpu_search_configs.py::test_config1_korf_linear_manhattan" -x -q > gpurun_out/r2_t4.log 2>&1
tests/cpp/bin/mma_microbench tmem > gpurun_out/r2_mma_tmem_contention.txt 2>&1
bash tests/search_host_sweep.sh > gpurun_out/host_sweep.log 2>&1
