"""Parity at BASELINE scale (VERDICT r1 "next" #1): every state checked, no
strided samples.

* BMLP1: the CUDA path against the independently pinned goldens
  (tests/golden/mlp_rc_*.npz: torch float64 layers + the reference's own
  compiled readout; make_golden_mlp.py), 100,000 reference random walks per
  model, H in {128, 256, 512, 1610}, E in {1, 2}.
* linear (the reference's own model): >= 1M reference random walks per domain
  against the reference's LinearModelBackend::evaluate compiled unchanged
  (oracle/_ref), run on every host thread.
* BMLP1 at 1M states against the oracle restatement.

Each test asserts zero flips and records how many (state, member) readouts
took the exact float64 replay (bida_gpu_exact_replays) in
gpurun_out/parity_scale.jsonl when that directory exists.
"""
from __future__ import annotations

import glob
import hashlib
import json
import os
import threading

import numpy as np
import pytest

import paper_2507_11916_b200 as bida
from oracle_lib import RC, STP3, STP4, Oracle, RefLib
from paper_2507_11916_b200.models import make_bmlp1

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
MLP_CASES = sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "mlp_rc_*.npz")))
THREADS = os.cpu_count() or 1


def record(**kw):
    out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out")
    if os.path.isdir(out):
        with open(os.path.join(out, "parity_scale.jsonl"), "a") as f:
            f.write(json.dumps(kw) + "\n")


@pytest.fixture(scope="module")
def ref():
    return RefLib()


@pytest.fixture(scope="module")
def golden_states(ref):
    z = np.load(os.path.join(GOLDEN, MLP_CASES[0] + ".npz"))
    lo, hi = (int(v) for v in z["walk_len"])
    packed = ref.random_walks(RC, int(z["n_states"]), lo, hi, int(z["state_seed"]))
    assert hashlib.sha256(packed.tobytes()).hexdigest() == str(z["states_sha256"])
    return packed


@pytest.mark.parametrize("name", MLP_CASES)
def test_mlp_matches_pinned_golden_100k(name, golden_states):
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    blob = make_bmlp1("rc", hidden=[int(h) for h in z["hidden"]], classes=int(z["classes"]),
                      ensemble=int(z["ensemble"]), seed=int(z["model_seed"]))
    assert hashlib.sha256(blob).hexdigest() == str(z["model_sha256"])
    with bida.MlpModelBackend("rc", blob, float(z["q"])) as be:
        h = be.evaluate(golden_states)
        replays = be.exact_replays()
    want = z["h"].astype(np.int32)
    flips = int((h != want).sum())
    record(test="mlp_pinned", case=name, states=len(h), flips=flips, exact_replays=replays,
           members=int(z["ensemble"]))
    assert flips == 0, f"{flips} flips against the pinned golden"


def _ref_linear_chunks(ref, d, W, q, packed, chunk=1 << 18):
    # the reference builds a float feature vector per state (1.9 KB for RC):
    # evaluate in chunks to bound host memory
    return np.concatenate([ref.linear_evaluate(d, W, q, packed[i:i + chunk], threads=THREADS)
                           for i in range(0, len(packed), chunk)])


@pytest.mark.parametrize("domain,E,C,q,wmax,lmax", [
    (RC, 1, 21, 0.5, 0.1, 30),
    (RC, 4, 21, 0.2, 1.0, 30),
    (STP4, 1, 64, 0.5, 0.1, 60),
    (STP3, 2, 32, 0.7, 0.5, 40),
])
def test_linear_1m_reference_walks_vs_reference(ref, domain, E, C, q, wmax, lmax):
    n = 1 << 20
    F = {RC: 480, STP4: 256, STP3: 81}[domain]
    W = np.random.default_rng(C * 31 + E).uniform(-wmax, wmax, (E, C, F)).astype(np.float32)
    packed = ref.random_walks(domain, n, 0, lmax, 7000 + domain + E)
    with bida.LinearModelBackend(domain, W, C, q) as be:
        h = be.evaluate(packed)
        replays = be.exact_replays()
    want = _ref_linear_chunks(ref, domain, W, q, packed)
    flips = int((h != want).sum())
    record(test="linear_1m_vs_reference", domain=domain, E=E, C=C, q=q, states=n, flips=flips,
           exact_replays=replays)
    assert flips == 0


def test_mlp_1m_reference_walks_vs_oracle(ref):
    n = 1 << 20
    blob = make_bmlp1("rc", hidden=[128, 128], classes=21, ensemble=1, seed=2507)
    packed = ref.random_walks(RC, n, 0, 30, 4242)
    with bida.MlpModelBackend("rc", blob, 0.5) as be:
        h = be.evaluate(packed)
        replays = be.exact_replays()
    want = Oracle().mlp_evaluate(blob, RC, 0.5, packed, threads=THREADS)
    flips = int((h != want).sum())
    record(test="mlp_1m_vs_oracle", hidden=[128, 128], states=n, flips=flips, exact_replays=replays)
    assert flips == 0


def test_ties_are_counted_as_replays():
    """Zero weights: a uniform softmax puts cum_k exactly on q = 0.5 -- every
    readout must take the exact replay, and the counter must say so."""
    W = np.zeros((1, 4, 480), np.float32)
    packed = bida.random_walks("rc", 1000, 0, 20, seed=3)
    with bida.LinearModelBackend("rc", W, 4, 0.5) as be:
        assert be.exact_replays() == 0
        be.evaluate(packed)
        assert be.exact_replays() == len(packed)


def test_errors_reported_to_the_offending_call_only():
    """Four threads share one handle; two submit batches holding a malformed
    state.  Each bad call raises, every good call returns OK with exact h
    (per-lane error words)."""
    rng = np.random.default_rng(5)
    W = rng.uniform(-0.1, 0.1, (1, 21, 480)).astype(np.float32)
    good = bida.random_walks("rc", 600, 0, 30, seed=6)
    bad = good.copy()
    bad["hi"][17] = np.uint64(0xFFFFFFFFFFFF)
    want = Oracle().linear_evaluate(RC, W, 0.5, good)
    res = {"good_ok": 0, "good_wrong": 0, "good_err": 0, "bad_err": 0, "bad_ok": 0}
    lock = threading.Lock()
    with bida.LinearModelBackend("rc", W, 21, 0.5) as be:
        def work(t):
            for _ in range(200):
                if t % 2:
                    try:
                        be.evaluate(bad)
                        key = "bad_ok"
                    except ValueError:
                        key = "bad_err"
                else:
                    try:
                        key = "good_ok" if (be.evaluate(good) == want).all() else "good_wrong"
                    except ValueError:
                        key = "good_err"
                with lock:
                    res[key] += 1
        ths = [threading.Thread(target=work, args=(t,)) for t in range(4)]
        for th in ths:
            th.start()
        for th in ths:
            th.join()
    assert res == {"good_ok": 400, "good_wrong": 0, "good_err": 0, "bad_err": 400, "bad_ok": 0}, res


def test_repeated_labels_use_dense_row_semantics(ref):
    """Rubik's states whose labels repeat or whose corner twist is 3 (never
    generated by the search, but encodable): the thread kernel's sort +
    deduplicate path must match the reference's dense one-hot row."""
    rng = np.random.default_rng(9)
    n = 4096
    packed = np.zeros(n, bida.instances.packed_dtype("rc"))
    lo = np.zeros(n, np.uint64)
    for p in range(8):
        lo |= rng.integers(0, 8, n).astype(np.uint64) << np.uint64(3 * p)
        lo |= rng.integers(0, 4, n).astype(np.uint64) << np.uint64(24 + 2 * p)
    for p in range(12):
        lo |= rng.integers(0, 2, n).astype(np.uint64) << np.uint64(40 + p)
    hi = np.zeros(n, np.uint64)
    for p in range(12):
        hi |= rng.integers(0, 12, n).astype(np.uint64) << np.uint64(4 * p)
    packed["lo"], packed["hi"] = lo, hi
    W = rng.uniform(-0.2, 0.2, (2, 21, 480)).astype(np.float32)
    with bida.LinearModelBackend("rc", W, 21, 0.5) as be:
        h, lg = be.evaluate_logits(packed)
    assert (h == ref.linear_evaluate(RC, W, 0.5, packed, threads=THREADS)).all()
    _, lo_ = Oracle().linear_evaluate(RC, W, 0.5, packed, want_logits=True)
    assert np.array_equal(lg.view(np.uint64), lo_.view(np.uint64))
