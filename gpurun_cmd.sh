set -x
timeout 900 python -m pytest tests/test_gpu_mlp.py -x -q 2>&1 | tail -15
timeout 300 python bench.py --workload rc-mlp-h1610 --steps 5 --warmup 3 --no-cpu-baseline --search-seconds 0 2>&1 | tail -1 | cut -c1-700
timeout 300 python bench.py --workload rc-mlp-h512 --steps 10 --warmup 3 --no-cpu-baseline --search-seconds 0 2>&1 | tail -1 | cut -c1-300
BIDA_MLP_FORCE_MODE=wide timeout 300 python bench.py --workload rc-mlp-h512 --steps 10 --warmup 3 --no-cpu-baseline --search-seconds 0 2>&1 | tail -1 | cut -c1-300
