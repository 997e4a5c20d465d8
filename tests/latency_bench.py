"""Per-call latency and throughput of bida_gpu_evaluate (host buffers) versus
batch size: the regime Batch IDA* runs in (batches of 1..8K states, SURVEY §7
hard part 2).  Not a pytest test; results are committed under profiles/.

    python tests/latency_bench.py --model mlp --hidden 128,128
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2507_11916_b200 as bida  # noqa: E402
from paper_2507_11916_b200.models import make_bmlp1  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="mlp", choices=["mlp", "linear"])
ap.add_argument("--hidden", default="128,128")
a = ap.parse_args()
if a.model == "mlp":
    be = bida.MlpModelBackend("rc", make_bmlp1("rc", hidden=[int(x) for x in a.hidden.split(",")], classes=21, seed=1), 0.5)
else:
    be = bida.LinearModelBackend("rc", np.random.default_rng(1).uniform(-0.1, 0.1, (1, 21, 480)).astype(np.float32), 21, 0.5)
packed = bida.random_walks("rc", 1 << 20, 0, 30, seed=2)
for B in [1, 8, 64, 512, 1024, 4096, 8192, 32768, 65536, 262144, 1048576]:
    x = np.ascontiguousarray(packed[:B])
    out = np.empty(B, np.int32)
    for _ in range(5):
        be.evaluate(x, out=out)
    reps = max(5, min(2000, int(2e6 // B)))
    t0 = time.perf_counter()
    for _ in range(reps):
        be.evaluate(x, out=out)
    dt = (time.perf_counter() - t0) / reps
    print(json.dumps({"model": a.model, "hidden": a.hidden, "batch": B, "us_per_call": dt * 1e6,
                      "evals_per_s": B / dt}), flush=True)
