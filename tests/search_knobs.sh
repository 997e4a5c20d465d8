#!/bin/bash
# Config-2 search knobs (work_num x flush timeout x shards, 12 searchers + 4 agents): gpurun_out/search_knobs.jsonl
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; rm -f gpurun_out/search_knobs.jsonl
python -c "from paper_2507_11916_b200.models import make_bmlp1; open('/tmp/h128.bmlp','wb').write(make_bmlp1('rc', hidden=[128, 128], classes=21, ensemble=1, seed=2507))"
for rep in 1 2; do for c in ${KNOBS:-128_25_16 64_25_16 256_25_16 128_10_16 128_50_16 128_25_8 128_25_32}; do
  IFS=_ read wn to sh <<< "$c"
  BIDA_EVAL_AGENTS=4 BIDA_EVAL_SHARDS=$sh timeout 200 tools/bin/bida_search_fast --domain rc --walks 1:14:14:2508 \
    --model mlp:/tmp/h128.bmlp --q 0.5 --table1-pdb 8 --pdb-build gpu --threads 12 --mode gpu --gpu-pdb \
    --work-num $wn --batch 16384 --timeout-us $to --time-limit 120 | python -c "import json,sys; r=json.loads(sys.stdin.readline()); print(json.dumps({'work_num':$wn,'timeout_us':$to,'shards':$sh, **{k:r[k] for k in ['status','generated','wall_s','nodes_per_s','mean_batch']}}))" >> gpurun_out/search_knobs.jsonl
done; done
