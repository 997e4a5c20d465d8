#!/bin/bash
# A/B of two search-driver builds on the config-2 instance (walk 14, seed 2508,
# 8-corner Table-1 PDB, 12 searchers + 4 agents): usage search_ab.sh exeA exeB [reps]
cd "$(dirname "$0")/.."
python - <<'PY'
from paper_2507_11916_b200.models import make_bmlp1
open("/tmp/h128.bmlp", "wb").write(make_bmlp1("rc", hidden=[128, 128], classes=21, ensemble=1, seed=2507))
PY
for rep in $(seq 1 ${3:-3}); do for exe in $1 $2; do
  BIDA_EVAL_AGENTS=${AGENTS:-4} BIDA_EVAL_SHARDS=16 timeout 200 tools/bin/$exe --domain rc --walks 1:14:14:2508 \
    --model mlp:/tmp/h128.bmlp --q 0.5 --table1-pdb 8 --pdb-build gpu --threads ${THREADS:-12} --mode gpu --gpu-pdb \
    --work-num ${WORK_NUM:-128} --batch 16384 --timeout-us ${TIMEOUT_US:-25} --time-limit 120 | python -c "import json,sys; r=json.loads(sys.stdin.readline()); print(json.dumps({'exe':'$exe', **{k:r[k] for k in ['status','generated','wall_s','nodes_per_s','mean_batch']}}))" >> gpurun_out/search_ab.jsonl
done; done
