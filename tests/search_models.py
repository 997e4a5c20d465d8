"""Config 4 / the paper's model-size table: Batch IDA*
nodes/s on one B200 as the network grows from the 0.2 MB to the 13.6 MB
anchor (H = 128 / 512 / 1610, two hidden layers), Rubik's walk-15, Table-1
mode (network evaluated for every node, 5-corner PDB guides the search), 16
host threads.  The CPU evaluator (oracle port) runs the same search for the
smaller nets.  Not a pytest test; -> profiles/."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2507_11916_b200.models import make_bmlp1  # noqa: E402

GPU_BIN = os.path.join(ROOT, "tools", "bin", "bida_search")
CPU_BIN = os.path.join(ROOT, "tests", "cpp", "bin", "search_parity")
n = min(16, os.cpu_count() or 16)
for hidden in ([128, 128], [512, 512], [1610, 1610]):
    model = f"/tmp/m{hidden[0]}.bmlp"
    open(model, "wb").write(make_bmlp1("rc", hidden=hidden, classes=21, seed=2507))
    mb = 4 * (480 * hidden[0] + hidden[0] * hidden[1] + hidden[1] * 21) / 1e6
    common = ["--domain", "rc", "--walks", "1:15:15:2508", "--model", "mlp:" + model, "--table1-pdb", "5",
              "--time-limit", "10", "--threads", str(n)]
    runs = [("gpu E=8", GPU_BIN, ["--mode", "gpu", "--gpu-pdb", "--evaluators", "8", "--work-num", "128",
                                  "--batch", "16384", "--timeout-us", "25"])]
    if hidden[0] <= 512:
        runs.append(("cpu-nn", CPU_BIN, ["--mode", "cpu", "--evaluators", str(n), "--work-num", "8", "--batch", "512",
                                         "--timeout-us", "200"]))
    for label, exe, extra in runs:
        out = subprocess.run([exe, *common, *extra], capture_output=True, text=True, timeout=600)
        for l in out.stdout.splitlines():
            if l.startswith("{"):
                r = json.loads(l)
                r.pop("iterations", None)
                r.update(label=label, hidden=hidden, fp32_mb=round(mb, 2))
                print(json.dumps(r), flush=True)
