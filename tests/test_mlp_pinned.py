"""BMLP1 parity pinned independently of the oracle (CPU).

tests/golden/mlp_rc_*.npz hold h-values produced by torch float64 layer
products plus the reference's own compiled readout
(LinearModelBackend::evaluate's softmax, quantile_class, ensemble_min;
batch_eval.hpp:98-168, heuristic.hpp:95-126) -- see make_golden_mlp.py.
Here the oracle's C restatement (oracle/bida_oracle.c, the checker every GPU
MLP test compares against) must reproduce them on the reference's own random
walks, 100,000 states per model (the GPU suite checks the CUDA path on the
same 100,000, tests/test_gpu_parity_scale.py)."""
from __future__ import annotations

import glob
import hashlib
import os

import numpy as np
import pytest

from oracle_lib import RC, Oracle, RefLib
from paper_2507_11916_b200.models import BMLP1, _one_hot, make_bmlp1

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CASES = sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "mlp_rc_*.npz")))


def load_case(name):
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    blob = make_bmlp1("rc", hidden=[int(h) for h in z["hidden"]], classes=int(z["classes"]),
                      ensemble=int(z["ensemble"]), seed=int(z["model_seed"]))
    assert hashlib.sha256(blob).hexdigest() == str(z["model_sha256"]), "model generator drifted"
    return z, blob


@pytest.fixture(scope="module")
def states():
    ref = RefLib()
    z = np.load(os.path.join(GOLDEN, CASES[0] + ".npz"))
    lo, hi = (int(v) for v in z["walk_len"])
    packed = ref.random_walks(RC, int(z["n_states"]), lo, hi, int(z["state_seed"]))
    assert hashlib.sha256(packed.tobytes()).hexdigest() == str(z["states_sha256"])
    return packed


def test_cases_present():
    assert len(CASES) == 8, CASES


@pytest.mark.parametrize("name", CASES)
def test_oracle_matches_pinned_golden(name, states):
    z, blob = load_case(name)
    n = len(states)
    E, C = int(z["ensemble"]), int(z["classes"])
    h, lg = Oracle().mlp_evaluate(blob, RC, float(z["q"]), states[:n], want_logits=True, E=E, Cc=C,
                                  threads=os.cpu_count() or 1)
    want = z["h"][:n].astype(np.int32)
    assert (h == want).all(), f"{int((h != want).sum())} of {n} h-values differ from the pinned golden"
    # logits of the head: the exact (double)acc * (double)out_scale
    k = min(n, len(z["acc_head"]))
    exact = z["acc_head"][:k].astype(np.float64) * z["out_scale"].astype(np.float64)[None, :, None]
    assert np.array_equal(lg[:k].view(np.uint64), exact.view(np.uint64))


def test_golden_accumulators_recompute(states):
    """The fixture's accumulators, recomputed with numpy int64 (a third
    implementation: models.forward_int) for the first 500 states."""
    from paper_2507_11916_b200.models import forward_int

    x = _one_hot(RC, states[:500])
    for name in CASES:
        z, blob = load_case(name)
        model = BMLP1.from_bytes(blob)
        for e, (layers, _s) in enumerate(model.members):
            acc = forward_int(layers, x)
            assert np.array_equal(acc, z["acc_head"][:500, e, :].astype(np.int64)), name


def test_reference_readout_encoding_is_exact():
    """ref_readout_scaled_logits (oracle/ref_harness.cpp) returns the
    reference's readout of (double)acc * (double)scale: checked against the
    reference's own quantile_class / ensemble_min applied to a softmax done
    here with math.exp (glibc, as std::exp) in the reference's order."""
    import math

    ref = RefLib()
    rng = np.random.default_rng(3)
    acc = rng.integers(-(2**31) + 1, 2**31 - 1, (300, 2, 21)).astype(np.int32)
    acc[:100] //= 1 << 20  # mostly moderate logits, some saturated
    scale = np.array([1.7e-7, -2.3e-8], np.float32)
    for q in (0.2, 0.5, 0.9):
        h = ref.readout_scaled_logits(RC, acc, scale, q)
        for i in range(len(acc)):
            est = []
            for m in range(2):
                lg = [float(a) * float(scale[m]) for a in acc[i, m]]
                mx = max(lg)
                ex = [math.exp(v - mx) for v in lg]
                z = 0.0
                for v in ex:
                    z += v
                est.append(ref.quantile_class(np.array([v / z for v in ex]), q))
            assert h[i] == ref.ensemble_min(est)
