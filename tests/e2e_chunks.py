"""End-to-end C-ABI rate (pinned host buffers, h128, 4M states per call) for
the current BIDA_GPU_CHUNK_LOG2, plus the H2D rate torch reaches when the same
bytes move as back-to-back chunks of that size on 4 streams (is the pipeline
bound by per-copy overhead?).  Not a test; one JSON line.

    BIDA_GPU_CHUNK_LOG2=18 python tests/e2e_chunks.py
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_11916_b200 as bida  # noqa: E402
from paper_2507_11916_b200.models import make_bmlp1  # noqa: E402

B = 1 << 22
k = int(os.environ.get("BIDA_GPU_CHUNK_LOG2", "18"))
packed = bida.random_walks_fast("rc", B, 0, 30, seed=5)
hp = torch.from_numpy(packed.view(np.uint8).copy()).pin_memory()
host = hp.numpy().view(packed.dtype)
out = torch.empty(B, dtype=torch.int32).pin_memory().numpy()
model = os.environ.get("E2E_MODEL", "h128")
if model == "linear":
    be = bida.LinearModelBackend("rc", np.random.default_rng(1).uniform(-0.1, 0.1, (1, 21, 480)).astype(np.float32), 21, 0.5)
else:
    hid = [1610, 1610] if model == "h1610" else [128, 128]
    be = bida.MlpModelBackend("rc", make_bmlp1("rc", hidden=hid, classes=21, seed=2507), 0.5)
with be:
    for _ in range(3):
        be.evaluate(host, out=out)
    t0 = time.perf_counter()
    reps = 20
    for _ in range(reps):
        be.evaluate(host, out=out)
    e2e = B * reps / (time.perf_counter() - t0)

# raw chunked H2D on 4 streams
dev = torch.empty(hp.numel(), dtype=torch.uint8, device="cuda")
streams = [torch.cuda.Stream() for _ in range(4)]
chunk = (1 << k) * 16
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(reps):
    for i, off in enumerate(range(0, hp.numel(), chunk)):
        with torch.cuda.stream(streams[i % 4]):
            dev[off:off + chunk].copy_(hp[off:off + chunk], non_blocking=True)
    torch.cuda.synchronize()
raw = hp.numel() * reps / (time.perf_counter() - t0) / 1e9
t0 = time.perf_counter()
for _ in range(reps):
    dev.copy_(hp, non_blocking=True)
    torch.cuda.synchronize()
whole = hp.numel() * reps / (time.perf_counter() - t0) / 1e9
print(json.dumps({"model": model, "direct": os.environ.get("BIDA_GPU_DIRECT", "1"), "chunk_log2": k, "e2e_evals_per_s": e2e, "e2e_h2d_gbs": e2e * 16 / 1e9,
                  "raw_chunked_h2d_gbs": raw, "raw_whole_h2d_gbs": whole}))
