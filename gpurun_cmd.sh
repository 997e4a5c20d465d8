timeout 900 python -m pytest tests/test_gpu_mlp.py -x -q -k "wide" 2>&1 | tail -3
for pr in 1 0; do echo "pair=$pr"; BIDA_MLP_WIDE_PAIR=$pr timeout 300 python bench.py --workload rc-mlp-h1610 --steps 5 --warmup 3 --no-cpu-baseline --search-seconds 0 2>&1 | tail -1 | cut -c1-100; done
for pr in 1 0; do echo "h512 pair=$pr"; BIDA_MLP_WIDE_PAIR=$pr BIDA_MLP_FORCE_MODE=wide timeout 300 python bench.py --workload rc-mlp-h512 --steps 5 --warmup 3 --no-cpu-baseline --search-seconds 0 2>&1 | tail -1 | cut -c1-100; done
for pr in 0 1; do BIDA_MLP_WIDE_PAIR=$pr timeout 120 python tests/trace_mlp.py --hidden 1610,1610 --tiles-per-cta 3 --warps 1,2 > gpurun_out/trace_wide7_$pr.txt 2>&1; done
