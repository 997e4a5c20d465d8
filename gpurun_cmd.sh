cd "$(dirname "$0")"
timeout 900 python -m pytest tests/test_gpu_mlp.py tests/test_gpu_linear.py tests/test_gpu_parity_scale.py -x -q > gpurun_out/r2_t7.log 2>&1
for w in rc-mlp-h128 rc-mlp-h256 rc-linear-e1-c21; do timeout 300 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline --search-seconds 0 --no-wide-leg --no-linear-leg --no-sweep 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(json.dumps({'workload':'$w','value':d['value'],'frac':d['roofline']['frac'],'e2e':d['e2e']['value']}))" >> gpurun_out/r2_quick_bench.jsonl; done
