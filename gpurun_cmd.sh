timeout 900 python -m pytest tests/test_gpu_mlp.py -x -q -k "every_schedule" 2>&1 | tail -2
for m in resident respair pair; do echo $m; BIDA_MLP_FORCE_MODE=$m timeout 300 python bench.py --workload rc-mlp-h128 --steps 10 --warmup 3 --no-cpu-baseline --search-seconds 0 --no-wide-leg 2>&1 | tail -1 | cut -c1-100; done
for m in respair pair; do echo $m h256; BIDA_MLP_FORCE_MODE=$m timeout 300 python bench.py --workload rc-mlp-h256 --steps 10 --warmup 3 --no-cpu-baseline --search-seconds 0 --no-wide-leg 2>&1 | tail -1 | cut -c1-100; done
