#!/bin/bash
# ThreadSanitizer runs of the ring evaluator + CB-DFS overlay (make -C tools tsan):
# CPU-only TableSim evaluators (--mode pdb, Table-1 semantics on a 4-corner PDB),
# several agent / shard / evaluator / batch settings.  Prints one line per run
# with the solve status and the number of TSAN reports (expected 0).
cd "$(dirname "$0")/.."
run() {
  local env="$1"; shift
  env $env TSAN_OPTIONS="halt_on_error=0" timeout 900 tools/bin/bida_search_fast_tsan "$@" > /tmp/tsan_o.txt 2> /tmp/tsan_e.txt
  local rc=$?
  local st=$(python -c "import json; r=json.loads(open('/tmp/tsan_o.txt').readline()); print(r['status'], r['cost'], r['generated'], r['batches'])" 2>/dev/null)
  echo "[$env] $* -> rc=$rc $st tsan_reports=$(grep -c 'WARNING: ThreadSanitizer' /tmp/tsan_e.txt)"
}
W="--domain rc --walks 2:8:8:11 --table1-pdb 4 --mode pdb --time-limit 300"
run "BIDA_EVAL_AGENTS=2 BIDA_EVAL_SHARDS=4" $W --threads 4 --work-num 8 --batch 64 --timeout-us 50
run "BIDA_EVAL_AGENTS=4 BIDA_EVAL_SHARDS=16" $W --threads 6 --work-num 16 --batch 256 --timeout-us 20
run "BIDA_EVAL_AGENTS=1 BIDA_EVAL_SHARDS=1" $W --threads 3 --work-num 4 --batch 16 --timeout-us 0
run "BIDA_EVAL_AGENTS=3 BIDA_EVAL_SHARDS=8" $W --threads 4 --work-num 8 --batch 128 --timeout-us -1 --evaluators 2
