"""Config 5's CPU thread-count sweep on one B200: Batch IDA* nodes/s vs
searcher threads for (a) GPU evaluators (network + PDB on the device),
(b) the same network on CPU evaluators (oracle port), (c) AIDA* with the PDB
only.  Rubik's walk-15, Table-1 mode.  Not a pytest test; -> profiles/."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2507_11916_b200.models import make_bmlp1  # noqa: E402

GPU_BIN = os.path.join(ROOT, "tools", "bin", "bida_search")
CPU_BIN = os.path.join(ROOT, "tests", "cpp", "bin", "search_parity")
model = "/tmp/m128.bmlp"
open(model, "wb").write(make_bmlp1("rc", hidden=[128, 128], classes=21, seed=2507))
ncpu = os.cpu_count() or 16
common = ["--domain", "rc", "--walks", "1:15:15:2508", "--model", "mlp:" + model, "--table1-pdb", "5",
          "--time-limit", "10"]
for n in sorted({2, 4, 8, 16, ncpu}):
    runs = [
        ("gpu", GPU_BIN, ["--mode", "gpu", "--gpu-pdb", "--evaluators", str(max(1, n // 2)), "--work-num", "128",
                          "--batch", "16384", "--timeout-us", "25"]),
        ("cpu-nn", CPU_BIN, ["--mode", "cpu", "--evaluators", str(n), "--work-num", "8", "--batch", "512",
                             "--timeout-us", "200"]),
        ("cpu-pdb-aidastar", CPU_BIN, ["--mode", "pdb", "--immediate"]),
    ]
    for label, exe, extra in runs:
        out = subprocess.run([exe, *common, "--threads", str(n), *extra], capture_output=True, text=True, timeout=600)
        for l in out.stdout.splitlines():
            if l.startswith("{"):
                r = json.loads(l)
                r.pop("iterations", None)
                r["label"] = label
                print(json.dumps(r), flush=True)
