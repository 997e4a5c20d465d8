cd "$(dirname "$0")"
rm -f gpurun_out/r2_chunk.jsonl
for rep in 1 2; do for k in 16 17 18 19 20; do
  BIDA_GPU_CHUNK_LOG2=$k timeout 300 python bench.py --workload rc-mlp-h128 --steps 20 --warmup 5 --no-cpu-baseline --search-seconds 0 --no-wide-leg --no-linear-leg --no-sweep 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(json.dumps({'chunk_log2':$k,'e2e':d['e2e']['value'],'pcie':d['e2e']['pcie']}))" >> gpurun_out/r2_chunk.jsonl
done; done
