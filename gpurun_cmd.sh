cd "$(dirname "$0")"
rm -f gpurun_out/host_sweep.jsonl
timeout 900 python bench.py > gpurun_out/r2_bench4.json 2> gpurun_out/r2_bench4.err
for th in 12 16; do for ag in 4; do
  BIDA_EVAL_AGENTS=$ag BIDA_EVAL_SHARDS=16 timeout 200 tools/bin/bida_search_fast --domain rc --walks 1:14:14:2508 \
    --model mlp:/tmp/h128.bmlp --q 0.5 --table1-pdb 8 --pdb-build gpu --threads $th --mode gpu --gpu-pdb \
    --work-num 128 --batch 16384 --timeout-us 25 --time-limit 120 | python -c "import json,sys; r=json.loads(sys.stdin.readline()); r.update(agents=$ag); print(json.dumps({k:r[k] for k in ['status','cost','generated','wall_s','nodes_per_s','mean_batch','threads','agents']}))" >> gpurun_out/host_sweep.jsonl
done; done
