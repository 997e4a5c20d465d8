"""Golden h-values for the BMLP1 MLP ensembles, pinned INDEPENDENTLY of the
oracle's C restatement (oracle/bida_oracle.c) and of the CUDA kernels.

The reference has no MLP, so BMLP1 is
pinned in two independent halves:

* layers: torch float64 matrix products on the CPU.  Every BMLP1 quantity is
  an integer of magnitude < 2^31, so float64 matmuls are exact in any
  summation order; requantisation is floor(acc / 2^shift) clamped to 0..255.
  This shares no code with the oracle's int32 triple loop.
* readout: the reference's OWN compiled LinearModelBackend::evaluate
  (batch_eval.hpp:98-105,148-168: max, exp, z, p = l / z; quantile_class and
  validate, heuristic.hpp:95-120; ensemble_min, heuristic.hpp:122-126) fed the
  exact output-layer logits (double)acc * (double)out_scale through
  ref_readout_scaled_logits (oracle/ref_harness.cpp explains the encoding).

States are the reference's own random walks (random_walk_instance,
instance.hpp:36-57, through oracle/_ref).  Each fixture stores h for
N_STATES states, the sha256 of the packed states and of the model blob (so a
test can regenerate both and prove they are the same), and the exact int32
output accumulators of the first N_ACC states.  Runs here only (needs
/root/reference); the GPU box reads the committed .npz files.

    python tests/golden/make_golden_mlp.py
"""
from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, ROOT)
from oracle_lib import RC, RefLib  # noqa: E402

from paper_2507_11916_b200.models import BMLP1, _one_hot, make_bmlp1  # noqa: E402

N_STATES = 100_000
N_ACC = 2_000
STATE_SEED = 2507_11916
# name: hidden widths, ensemble size, q, model seed
CASES = {
    "mlp_rc_h128_e1": ([128, 128], 1, 0.5, 5),
    "mlp_rc_h128_e2": ([128, 128], 2, 0.3, 6),
    "mlp_rc_h256_e1": ([256, 256], 1, 0.5, 7),
    "mlp_rc_h256_e2": ([256, 256], 2, 0.7, 8),
    "mlp_rc_h512_e1": ([512, 512], 1, 0.5, 9),
    "mlp_rc_h512_e2": ([512, 512], 2, 0.5, 10),
    "mlp_rc_h1610_e1": ([1610, 1610], 1, 0.5, 2507),
    "mlp_rc_h1610_e2": ([1610, 1610], 2, 0.9, 12),
}


def states_sha(packed: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(packed).tobytes()).hexdigest()


def torch_accumulators(model: BMLP1, x: np.ndarray, chunk: int = 20_000) -> np.ndarray:
    """Output accumulators [n][E][C] (int32) by float64 torch matmuls."""
    torch.set_num_threads(os.cpu_count() or 1)
    n = len(x)
    out = np.zeros((n, len(model.members), model.C), np.int32)
    for e, (layers, _scale) in enumerate(model.members):
        Ws = [torch.from_numpy(ly.W.astype(np.float64)) for ly in layers]
        bs = [torch.from_numpy(ly.bias.astype(np.float64)) for ly in layers]
        for i0 in range(0, n, chunk):
            a = torch.from_numpy(x[i0:i0 + chunk].astype(np.float64))
            for li, ly in enumerate(layers):
                acc = a @ Ws[li].T + bs[li]
                assert float(acc.abs().max()) < 2.0**31
                if li < len(layers) - 1:
                    a = torch.clamp(torch.floor(acc / float(1 << ly.shift)), 0, 255)
                else:
                    out[i0:i0 + chunk, e, :] = acc.numpy().astype(np.int32)
    return out


def main() -> None:
    ref = RefLib()
    packed = ref.random_walks(RC, N_STATES, 0, 30, STATE_SEED)
    x = _one_hot(RC, packed)
    sha_states = states_sha(packed)
    for name, (hidden, E, q, seed) in CASES.items():
        t0 = time.time()
        blob = make_bmlp1("rc", hidden=hidden, classes=21, ensemble=E, seed=seed)
        model = BMLP1.from_bytes(blob)
        acc = torch_accumulators(model, x)
        scale = np.array([s for _, s in model.members], np.float32)
        h = ref.readout_scaled_logits(RC, acc, scale, q, threads=os.cpu_count() or 1)
        np.savez_compressed(
            os.path.join(HERE, name + ".npz"), domain=RC, hidden=np.array(hidden), ensemble=E, classes=21,
            q=q, model_seed=seed, model_sha256=hashlib.sha256(blob).hexdigest(), state_seed=STATE_SEED,
            n_states=N_STATES, walk_len=np.array([0, 30]), states_sha256=sha_states, h=h.astype(np.uint8),
            acc_head=acc[:N_ACC], out_scale=scale)
        print(f"{name}: {time.time() - t0:.1f} s, h histogram {np.bincount(h).tolist()}", flush=True)


if __name__ == "__main__":
    main()
