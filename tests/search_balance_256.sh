#!/bin/bash
# searcher threads vs agents with 256 subtrees / 15 us (config-2 instance): gpurun_out/search_balance2.jsonl
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; rm -f gpurun_out/search_balance2.jsonl
python -c "from paper_2507_11916_b200.models import make_bmlp1; open('/tmp/h128.bmlp','wb').write(make_bmlp1('rc', hidden=[128, 128], classes=21, ensemble=1, seed=2507))"
for rep in 1 2; do for c in 12_4 13_3 11_5 14_2; do
  t=${c%_*}; a=${c#*_}
  BIDA_EVAL_AGENTS=$a BIDA_EVAL_SHARDS=16 timeout 200 tools/bin/bida_search_fast --domain rc --walks 1:14:14:2508 \
    --model mlp:/tmp/h128.bmlp --q 0.5 --table1-pdb 8 --pdb-build gpu --threads $t --mode gpu --gpu-pdb \
    --work-num 256 --batch 16384 --timeout-us 15 --time-limit 120 | python -c "import json,sys; r=json.loads(sys.stdin.readline()); print(json.dumps({'threads':$t,'agents':$a, **{k:r[k] for k in ['status','generated','wall_s','nodes_per_s','mean_batch']}}))" >> gpurun_out/search_balance2.jsonl
done; done
