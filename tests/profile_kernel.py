"""Small driver for ncu --set full captures of one evaluator kernel (faster to
set up than bench.py): a device-resident batch, W warm-up launches, then the
profiled launches.  Not a test; prints nothing but a status line.

    python tests/profile_kernel.py --model mlp --hidden 128,128 --n 1048576 --launches 4
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_11916_b200 as bida  # noqa: E402
from paper_2507_11916_b200.models import make_bmlp1  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="mlp", choices=["mlp", "linear"])
ap.add_argument("--hidden", default="128,128")
ap.add_argument("--classes", type=int, default=21)
ap.add_argument("--ensemble", type=int, default=1)
ap.add_argument("--n", type=int, default=1 << 20)
ap.add_argument("--launches", type=int, default=4)
a = ap.parse_args()
packed = bida.random_walks("rc", a.n, 0, 30, seed=1)
d_in = torch.from_numpy(packed.view(np.uint8).copy()).cuda()
d_h = torch.empty(a.n, dtype=torch.int32, device="cuda")
if a.model == "mlp":
    hidden = [int(x) for x in a.hidden.split(",")]
    be = bida.MlpModelBackend("rc", make_bmlp1("rc", hidden=hidden, classes=a.classes, ensemble=a.ensemble, seed=2507), 0.5)
else:
    W = np.random.default_rng(2507).uniform(-0.1, 0.1, (a.ensemble, a.classes, 480)).astype(np.float32)
    be = bida.LinearModelBackend("rc", W, a.classes, 0.5)
for _ in range(a.launches):
    be.evaluate_device(d_in, d_h)
torch.cuda.synchronize()
be.status()
print("ok", a.model, a.hidden, a.n, be.launch_count())
