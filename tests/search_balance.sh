#!/bin/bash
# searcher threads vs agents on a 16-core host (config-2 instance, walk 14 seed 2508)
cd "$(dirname "$0")/.."
python - <<'PY'
from paper_2507_11916_b200.models import make_bmlp1
open("/tmp/h128.bmlp", "wb").write(make_bmlp1("rc", hidden=[128, 128], classes=21, ensemble=1, seed=2507))
PY
for cfg in "12 4" "11 5" "10 6" "8 8" "14 2" "13 3"; do set -- $cfg
  BIDA_EVAL_AGENTS=$2 BIDA_EVAL_SHARDS=16 timeout 200 tools/bin/bida_search_fast --domain rc --walks 1:14:14:2508 \
    --model mlp:/tmp/h128.bmlp --q 0.5 --table1-pdb 8 --pdb-build gpu --threads $1 --mode gpu --gpu-pdb \
    --work-num 128 --batch 16384 --timeout-us 25 --time-limit 120 | python -c "import json,sys; r=json.loads(sys.stdin.readline()); print(json.dumps({'threads':$1,'agents':$2, **{k:r[k] for k in ['status','generated','wall_s','nodes_per_s','mean_batch']}}))" >> gpurun_out/search_balance.jsonl
done
