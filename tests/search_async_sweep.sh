#!/bin/bash
# Ring agents with the asynchronous backend path (several batches in flight per
# agent) vs synchronous calls (BIDA_EVAL_INFLIGHT=1), config-2 instance (walk 14,
# seed 2508, 8-corner Table-1 PDB).  JSON lines -> gpurun_out/async_sweep.jsonl
cd "$(dirname "$0")/.."
python - <<'PY'
from paper_2507_11916_b200.models import make_bmlp1
open("/tmp/h128.bmlp", "wb").write(make_bmlp1("rc", hidden=[128, 128], classes=21, ensemble=1, seed=2507))
PY
for th in 12 16; do for ag in 1 2 4; do for inf in 1 0; do
  BIDA_EVAL_INFLIGHT=$inf BIDA_EVAL_AGENTS=$ag BIDA_EVAL_SHARDS=16 timeout 200 tools/bin/bida_search_fast --domain rc --walks 1:14:14:2508 \
    --model mlp:/tmp/h128.bmlp --q 0.5 --table1-pdb 8 --pdb-build gpu --threads $th --mode gpu --gpu-pdb \
    --work-num 128 --batch 16384 --timeout-us 25 --time-limit 120 | python -c "import json,sys; r=json.loads(sys.stdin.readline()); r.update(agents=$ag, inflight_env=$inf); print(json.dumps({k:r[k] for k in ['status','cost','generated','wall_s','nodes_per_s','mean_batch','threads','agents','inflight_env']}))" >> gpurun_out/async_sweep.jsonl
done; done; done
