"""Batch IDA* nodes/s sweep over evaluator count and flush timeout (Rubik's,
Table-1 mode with the device PDB).  Not a pytest test; results -> profiles/."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
BIN = os.path.join(ROOT, "tests", "cpp", "bin", "search_parity")
from paper_2507_11916_b200.models import make_bmlp1  # noqa: E402

model = "/tmp/m128.bmlp"
open(model, "wb").write(make_bmlp1("rc", hidden=[128, 128], classes=21, seed=2507))
threads = int(sys.argv[1]) if len(sys.argv) > 1 else 16
for E in (1, 2, 4, 8):
    for to in (0, 25, 100):
        for k in (32, 128):
            cmd = [BIN, "--domain", "rc", "--walks", "1:15:15:2508", "--model", "mlp:" + model, "--mode", "gpu",
                   "--table1-pdb", "5", "--gpu-pdb", "--threads", str(threads), "--time-limit", "15",
                   "--evaluators", str(E), "--work-num", str(k), "--batch", "16384", "--timeout-us", str(to)]
            out = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
            for l in out.stdout.splitlines():
                if l.startswith("{"):
                    r = json.loads(l)
                    r.pop("iterations", None)
                    print(json.dumps(r), flush=True)
