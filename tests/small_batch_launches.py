"""Driver for an ncu launch list of small-batch evaluations (device-resident
batches of 1..4096 states, linear and BMLP1 h128): the kernel durations
behind profiles/r2_latency_breakdown_*.jsonl.  Not a test."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_11916_b200 as bida  # noqa: E402
from paper_2507_11916_b200.models import make_bmlp1  # noqa: E402

d_in = bida.random_walks_device("rc", 4096, 0, 30, seed=1)
d_h = torch.empty(4096, dtype=torch.int32, device="cuda")
W = np.random.default_rng(1).uniform(-0.1, 0.1, (1, 21, 480)).astype(np.float32)
for be in (bida.LinearModelBackend("rc", W, 21, 0.5),
           bida.MlpModelBackend("rc", make_bmlp1("rc", hidden=[128, 128], classes=21, seed=2507), 0.5)):
    for n in (1, 64, 1024, 4096):
        for _ in range(3):
            be.evaluate_device(d_in, d_h, n=n)
    torch.cuda.synchronize()
    be.status()
print("ok")
