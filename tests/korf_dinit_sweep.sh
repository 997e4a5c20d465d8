#!/bin/bash
# Config 1 (Korf #9 #5 #2 #6 #8, linear-Manhattan C=72): GPU Batch IDA* (ring +
# CB-DFS overlay) against the reference's CPU AIDA* (LinearModelBackend, one
# subtree per thread) at fixed d_init (work generation depth, search.hpp:61-79).
# JSON lines -> gpurun_out/korf_dinit.jsonl
cd "$(dirname "$0")/.."
python - <<'PY'
import sys, numpy as np
sys.path.insert(0, "tests")
from oracle_lib import manhattan_linear_weights
import paper_2507_11916_b200 as bida
g = np.load("tests/golden/instances.npz")
open("/tmp/bida_korf10.txt", "w").write("".join("stp 4 " + " ".join(str((int(v) >> (4 * c)) & 15) for c in range(16)) + "\n" for v in g["korf10"]))
open("/tmp/bida_man4.blin", "wb").write(bida.blin1_bytes("stp4", manhattan_linear_weights(4, 72, 4.0), 72))
PY
T=$(nproc)
EXTRACT="import json,sys; r=json.loads(sys.stdin.readline()); print(json.dumps({k:r.get(k) for k in ['instance','mode','status','cost','generated','wall_s','nodes_per_s','mean_batch','thresholds','iterations','work_num','evaluators']}))"
for k in 8 4 1 5 7; do for d in ${DINITS:-10 12 14}; do
  BIDA_EVAL_AGENTS=2 BIDA_EVAL_SHARDS=16 timeout 300 tools/bin/bida_search_fast --domain stp4 --instances /tmp/bida_korf10.txt \
    --model linear:/tmp/bida_man4.blin --q 0.5 --first $k --count 1 --threads $T --mode gpu --work-num ${WORK_NUM:-64} --batch 8192 \
    --timeout-us 20 --d-init $d --time-limit 240 | python -c "$EXTRACT" | sed "s/^{/{\"d_init\": $d, \"side\": \"gpu\", \"work_num_gpu\": ${WORK_NUM:-64}, /" >> gpurun_out/korf_dinit.jsonl
  timeout 300 tools/bin/bida_search --domain stp4 --instances /tmp/bida_korf10.txt \
    --model linear:/tmp/bida_man4.blin --q 0.5 --first $k --count 1 --threads $T --mode cpu --immediate --work-num 1 \
    --d-init $d --time-limit 240 | python -c "$EXTRACT" | sed "s/^{/{\"d_init\": $d, \"side\": \"cpu_aidastar\", /" >> gpurun_out/korf_dinit.jsonl
done; done
