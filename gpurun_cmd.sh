cd "$(dirname "$0")"
python - <<'PY'
from paper_2507_11916_b200.models import make_bmlp1
open("/tmp/h128.bmlp","wb").write(make_bmlp1("rc", hidden=[128,128], classes=21, ensemble=1, seed=2507))
PY
for exe in bida_search_ring bida_search_fast bida_search_ring bida_search_fast; do
  BIDA_EVAL_AGENTS=4 BIDA_EVAL_SHARDS=16 timeout 120 tools/bin/$exe --domain rc --walks 1:15:15:2508 --model mlp:/tmp/h128.bmlp --mode gpu --gpu-pdb --table1-pdb 5 --threads 16 --work-num 128 --batch 16384 --timeout-us 25 --time-limit 10 | python -c "import json,sys; r=json.loads(sys.stdin.readline()); print('$exe', r['status'], round(r['nodes_per_s']/1e6,2), 'M nodes/s', r['mean_batch'])" >> gpurun_out/r2_fast_vs_ring.txt
done
timeout 2400 python tests/search_screen.py --lengths 14,15,16 --seeds 4 --gpu-limit 40 --cpu-limit 100 > gpurun_out/r2_screen.log 2>&1
