"""Prints the clock64 timeline of CTA 0 of the MLP kernel (debug; not a test).
    python tests/trace_mlp.py --hidden 128,128 --tiles-per-cta 8"""
import argparse
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["BIDA_GPU_TRACE"] = "1"  # the diagnostic library (built in the build container: build(trace=True))
import paper_2507_11916_b200 as bida  # noqa: E402
from paper_2507_11916_b200 import _native  # noqa: E402
from paper_2507_11916_b200.models import make_bmlp1  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--hidden", default="128,128")
ap.add_argument("--tiles-per-cta", type=int, default=8)
ap.add_argument("--warps", default="1,2,6")
a = ap.parse_args()
hidden = [int(x) for x in a.hidden.split(",")]
n = 148 * 128 * a.tiles_per_cta
packed = bida.random_walks("rc", n, 0, 30, seed=1)
d_in = torch.from_numpy(packed.view(np.uint8).copy()).cuda()
d_h = torch.empty(n, dtype=torch.int32, device="cuda")
be = bida.MlpModelBackend("rc", make_bmlp1("rc", hidden=hidden, classes=21, seed=3), 0.5)
slots = _native.lib().bida_gpu_trace_slots()
buf = torch.zeros(32 * slots, dtype=torch.int64, device="cuda")
be.evaluate_device(d_in, d_h)  # warm
torch.cuda.synchronize()
_native.check(_native.lib().bida_gpu_debug_trace(be._h, C.c_void_p(buf.data_ptr())))
be.evaluate_device(d_in, d_h)
torch.cuda.synchronize()
t = buf.cpu().numpy().reshape(32, slots)
t0 = min(int(x) >> 8 for x in t.ravel() if x and (int(x) & 0xFF) != 90)
names = {10: "mma wait act L", 20: "mma got act L", 30: "mma commit L", 40: "epi encode", 41: "epi enc done",
         50: "epi wait d L", 60: "epi got d L", 70: "epi hidden done L", 80: "epi readout done",
         84: "tile top", 85: "next state load issued", 86: "tile setup done"}
for w in [int(x) for x in a.warps.split(",")]:
    print(f"--- warp {w}")
    for x in t[w]:
        if not x:
            break
        tag = int(x) & 0xFF
        base = max(k for k in names if k <= tag)
        if tag == 90:
            print(f"{'':9s}  (stage waits in this chunk: {int(x) >> 8} cycles)")
            continue
        if tag in (81, 82, 83):
            print(f"{(int(x) >> 8) - t0:9d}  readout mark {tag}")
            continue
        print(f"{(int(x) >> 8) - t0:9d}  {names[base]}{tag - base if base not in (40, 41, 80, 84, 85, 86) else ''}")
