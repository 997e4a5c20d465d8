cd $GRAFT_REPO_ROOT
python -c "from paper_2507_11916_b200.models import make_bmlp1; open('/tmp/ra.bmlp','wb').write(make_bmlp1('rc', hidden=[128,128], classes=21, seed=2507))"
for rep in 1 2 3; do for KS in 2:8 4:16 8:16 4:8; do K=${KS%:*}; S=${KS#*:}
  BIDA_EVAL_AGENTS=$K BIDA_EVAL_SHARDS=$S timeout 120 tools/bin/bida_search_ring --domain rc --walks 1:15:15:2508 \
    --model mlp:/tmp/ra.bmlp --table1-pdb 5 --time-limit 8 --mode gpu --gpu-pdb --work-num 128 --threads 16 \
    --evaluators 1 --batch 16384 --timeout-us 25 | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        r = json.loads(l); r.pop('iterations', None); r.update(agents=$K, shards=$S, rep=$rep); print(json.dumps(r))"
done; done
