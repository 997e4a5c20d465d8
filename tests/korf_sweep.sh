#!/bin/bash
# Config-1 (Korf #9, linear-Manhattan C=72) GPU Batch IDA* knob sweep: work_num,
# flush timeout, agents.  One JSON line per run into gpurun_out/korf_sweep.jsonl.
cd "$(dirname "$0")/.."
python - <<'PY'
import sys, os, numpy as np
sys.path.insert(0, "tests")
from oracle_lib import manhattan_linear_weights
import paper_2507_11916_b200 as bida
g = np.load("tests/golden/instances.npz")
open("/tmp/bida_korf10.txt", "w").write("".join("stp 4 " + " ".join(str((int(v) >> (4 * c)) & 15) for c in range(16)) + "\n" for v in g["korf10"]))
open("/tmp/bida_man4.blin", "wb").write(bida.blin1_bytes("stp4", manhattan_linear_weights(4, 72, 4.0), 72))
PY
T=$(nproc)
for wn in 64 256 1024; do for to in 0 20; do for ag in 2 4; do
  BIDA_EVAL_AGENTS=$ag BIDA_EVAL_SHARDS=16 timeout 120 tools/bin/bida_search_fast --domain stp4 --instances /tmp/bida_korf10.txt \
    --model linear:/tmp/bida_man4.blin --q 0.5 --first 8 --count 1 --threads $T --mode gpu --work-num $wn --batch 8192 \
    --timeout-us $to --time-limit 100 | python -c "import json,sys; r=json.loads(sys.stdin.readline()); r.update(agents=$ag); print(json.dumps({k:r[k] for k in ['status','cost','generated','wall_s','nodes_per_s','mean_batch','work_num','timeout_us','agents']}))" >> gpurun_out/korf_sweep.jsonl
done; done; done
