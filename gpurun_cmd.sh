#!/bin/bash
cd "$(dirname "$0")"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_graphs.py tests/test_gpu_async.py tests/test_gpu_pdb.py tests/test_gpu_linear.py tests/test_gpu_mlp.py -q -x > gpurun_out/graphs_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/graphs_tests.log
python - <<'PY'
from paper_2507_11916_b200.models import make_bmlp1
open("/tmp/h128.bmlp", "wb").write(make_bmlp1("rc", hidden=[128, 128], classes=21, ensemble=1, seed=2507))
PY
for g in 0 1; do
  BIDA_GPU_GRAPHS=$g timeout 120 tests/cpp/bin/latency_breakdown /tmp/h128.bmlp mlp > gpurun_out/lat_graph$g.jsonl 2>&1
  BIDA_GPU_GRAPHS=$g timeout 120 tests/cpp/bin/latency_breakdown "" linear > gpurun_out/lat_lin_graph$g.jsonl 2>&1
done
rm -f gpurun_out/search_graph_ab.jsonl
for rep in 1 2 3; do for g in 0 1; do
  BIDA_GPU_GRAPHS=$g BIDA_EVAL_AGENTS=4 BIDA_EVAL_SHARDS=16 timeout 200 tools/bin/bida_search_fast --domain rc --walks 1:14:14:2508 \
    --model mlp:/tmp/h128.bmlp --q 0.5 --table1-pdb 8 --pdb-build gpu --threads 12 --mode gpu --gpu-pdb \
    --work-num 128 --batch 16384 --timeout-us 25 --time-limit 120 | python -c "import json,sys; r=json.loads(sys.stdin.readline()); print(json.dumps({'graphs':$g, **{k:r[k] for k in ['status','generated','wall_s','nodes_per_s','mean_batch']}}))" >> gpurun_out/search_graph_ab.jsonl
done; done
