#!/bin/bash
# Ring evaluator agents/shards sweep at one evaluator on one B200 (-> profiles/r1_search_ring_agents.jsonl).
# Same search as bench.py's search legs: Rubik's walk-15, BMLP1 480-128-128-21 + 5-corner PDB on the device.
cd "$(dirname "$0")/.."
python -c "from paper_2507_11916_b200.models import make_bmlp1; open('/tmp/ra.bmlp','wb').write(make_bmlp1('rc', hidden=[128,128], classes=21, seed=2507))"
T=$(python -c "import os; print(len(os.sched_getaffinity(0)))")
for K in 1 2 4; do for S in 8 16; do for W in 128 256; do
  BIDA_EVAL_AGENTS=$K BIDA_EVAL_SHARDS=$S timeout 120 tools/bin/bida_search_ring --domain rc --walks 1:15:15:2508 \
    --model mlp:/tmp/ra.bmlp --table1-pdb 5 --time-limit 8 --mode gpu --gpu-pdb --work-num $W --threads $T \
    --evaluators 1 --batch 16384 --timeout-us 25 | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        r = json.loads(l); r.pop('iterations', None); r.update(agents=$K, shards=$S); print(json.dumps(r))"
done; done; done
