"""A/B timing of one library build (BIDA_GPU_LIB selects it) on the fused MLP
schedules: device evals/s over rotating device-resident batches (CUDA events),
plus a bit-exactness check of a sample against the oracle.  Not a test; one
JSON line per model.

    BIDA_GPU_LIB=paper_2507_11916_b200/_lib/libbida_gpu_g3.so python tests/mlp_ab.py --tag g3
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2507_11916_b200 as bida  # noqa: E402
from paper_2507_11916_b200.models import make_bmlp1  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--tag", default=os.environ.get("BIDA_GPU_LIB", "default"))
ap.add_argument("--models", default="128,128;256,256;512,512;128,128,128")
ap.add_argument("--n", type=int, default=1 << 22)
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--check", type=int, default=65536)
a = ap.parse_args()

bufs = [bida.random_walks_device("rc", a.n, 0, 30, seed=100 + i) for i in range(4)]
d_h = torch.empty(a.n, dtype=torch.int32, device="cuda")
from oracle_lib import RC, Oracle  # noqa: E402

orc = Oracle()
for spec in a.models.split(";"):
    hidden = [int(x) for x in spec.split(",")]
    blob = make_bmlp1("rc", hidden=hidden, classes=21, ensemble=1, seed=2507)
    with bida.MlpModelBackend("rc", blob, 0.5) as be:
        for i in range(3):
            be.evaluate_device(bufs[i % 4], d_h)
        torch.cuda.synchronize()
        st = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for i in range(a.reps):
            be.evaluate_device(bufs[i % 4], d_h)
        e1.record(st)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        sample = bufs[0][: a.check * 16].cpu().numpy().view(bida.instances.packed_dtype("rc"))
        got = be.evaluate(sample)
        want = orc.mlp_evaluate(blob, RC, 0.5, sample, threads=16)
        print(json.dumps({"tag": a.tag, "hidden": hidden, "n": a.n, "ms": round(ms, 4),
                          "evals_per_s": a.n / ms * 1e3, "flips": int((got != want).sum())}), flush=True)
