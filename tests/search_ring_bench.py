"""SURVEY §8(f) row 1 measurement on one B200: Batch IDA* nodes/s with the
reference's Evaluator (tools/bin/bida_search) vs the ring evaluator
(tools/bin/bida_search_ring), both with GpuBackend (network + PDB on the
device), swept over evaluators per GPU and submit-ring shards per evaluator.  Rubik's
walk-15, Table-1 mode, BMLP1 480-128-128-21.  Not a pytest test; -> profiles/."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2507_11916_b200.models import make_bmlp1  # noqa: E402

secs = sys.argv[1] if len(sys.argv) > 1 else "8"
model = "/tmp/ring128.bmlp"
open(model, "wb").write(make_bmlp1("rc", hidden=[128, 128], classes=21, seed=2507))
ncpu = len(os.sched_getaffinity(0))
common = ["--domain", "rc", "--walks", "1:15:15:2508", "--model", "mlp:" + model, "--table1-pdb", "5",
          "--time-limit", secs, "--mode", "gpu", "--gpu-pdb", "--work-num", "128", "--threads", str(ncpu)]
runs = []
if len(sys.argv) > 2 and sys.argv[2] == "threads":
    # config 5's CPU thread sweep with one ring evaluator (the one-evaluator-per-GPU mapping)
    for n in sorted({2, 4, 8, 16, ncpu}):
        common[common.index("--threads") + 1] = str(n)
        for impl, exe, K, S in (("reference", "bida_search", 1, 1), ("ring", "bida_search_ring", 2, 8)):
            out = subprocess.run([os.path.join(ROOT, "tools", "bin", exe), *common, "--evaluators", "1", "--batch",
                                  "16384", "--timeout-us", "25"], capture_output=True, text=True, timeout=600,
                                 env={**os.environ, "BIDA_EVAL_AGENTS": str(K), "BIDA_EVAL_SHARDS": str(S)})
            for l in out.stdout.splitlines():
                if l.startswith("{"):
                    r = json.loads(l)
                    r.pop("iterations", None)
                    r.update(impl=impl, agents=K, shards=S, host_threads=ncpu)
                    print(json.dumps(r), flush=True)
    sys.exit(0)
for E in (1, 2, 8):
    runs.append(("reference", "bida_search", E, 1, 1, 16384, 25))
    for S in (1, 4, 8):
        runs.append(("ring", "bida_search_ring", E, 2, S, 16384, 25))
    runs.append(("ring", "bida_search_ring", E, 2, 4, 4096, 0))
for impl, exe, E, K, S, B, t in runs:
    out = subprocess.run([os.path.join(ROOT, "tools", "bin", exe), *common, "--evaluators", str(E), "--batch", str(B),
                          "--timeout-us", str(t)], capture_output=True, text=True, timeout=600,
                         env={**os.environ, "BIDA_EVAL_AGENTS": str(K), "BIDA_EVAL_SHARDS": str(S)})
    rows = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    if out.returncode or not rows:
        print(json.dumps({"impl": impl, "evaluators": E, "agents": K, "shards": S, "error": out.stderr[-300:]}), flush=True)
        continue
    r = rows[0]
    r.pop("iterations", None)
    r.update(impl=impl, agents=K, shards=S, host_threads=ncpu)
    print(json.dumps(r), flush=True)
