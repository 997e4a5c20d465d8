#!/bin/bash
# Config 1 GPU-side knobs (Korf #5, d_init 14, linear-Manhattan C=72): agents x
# work_num x flush timeout x searcher threads.  JSON lines -> gpurun_out/korf_tune.jsonl
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
EXTRACT="import json,sys; r=json.loads(sys.stdin.readline()); print(json.dumps({k:r.get(k) for k in ['status','cost','generated','wall_s','nodes_per_s','mean_batch']}))"
for cfg in ${KORF_CFGS:-2_64_20_16 4_64_20_16 2_128_20_16 2_256_20_16 4_256_20_16 2_64_10_16 2_64_40_16 4_128_10_14 2_128_10_14 6_128_10_12}; do
  IFS=_ read a wn to th <<< "$cfg"
  BIDA_EVAL_AGENTS=$a BIDA_EVAL_SHARDS=16 timeout 300 tools/bin/bida_search_fast --domain stp4 --instances /tmp/bida_korf10.txt \
    --model linear:/tmp/bida_man4.blin --q 0.5 --first ${KORF_FIRST:-5} --count 1 --threads $th --mode gpu --work-num $wn --batch 8192 \
    --timeout-us $to --d-init 14 --time-limit 120 | python -c "$EXTRACT" | sed "s/^{/{\"first\": ${KORF_FIRST:-5}, \"agents\": $a, \"work_num\": $wn, \"timeout_us\": $to, \"threads\": $th, /" >> gpurun_out/korf_tune.jsonl
done
