cd "$(dirname "$0")"
rm -f gpurun_out/r2_ab.jsonl
for rep in 1 2 3; do for lib in libbida_gpu.so libbida_gpu_prev.so; do for w in rc-mlp-h128 rc-linear-e1-c21; do
  BIDA_GPU_LIB=$PWD/paper_2507_11916_b200/_lib/$lib timeout 300 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline --search-seconds 0 --no-wide-leg --no-linear-leg --no-sweep 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(json.dumps({'lib':'$lib','workload':'$w','value':d['value'],'kern_ms':d['kernel_ms_avg']}))" >> gpurun_out/r2_ab.jsonl
done; done; done
