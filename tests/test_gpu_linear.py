"""GPU parity of the fused linear evaluator against the reference's golden
vectors and the oracle, through the C-ABI.  Bar: h bit-exact on every state,
float64 logits bit-exact (same operations, same order)."""
import glob
import os

import numpy as np
import pytest

import paper_2507_11916_b200 as bida
from oracle_lib import FEATURES, RC, STP2, STP3, STP4, Oracle, manhattan_linear_weights

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def orc():
    return Oracle()


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLDEN, "linear_*.npz"))))
def test_golden_h_bit_exact(path):
    g = np.load(path)
    d = int(g["domain"])
    W = g["W"]
    with bida.LinearModelBackend(d, W, W.shape[1], float(g["q"])) as be:
        h = be.evaluate(g["packed"])
    assert (h == g["h"]).all(), f"{(h != g['h']).sum()} flips"


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLDEN, "linear_*.npz"))))
def test_logits_bit_exact_vs_oracle(orc, path):
    g = np.load(path)
    d = int(g["domain"])
    W = g["W"]
    with bida.LinearModelBackend(d, W, W.shape[1], float(g["q"])) as be:
        h, lg = be.evaluate_logits(g["packed"])
    ho, lo = orc.linear_evaluate(d, W, float(g["q"]), g["packed"], want_logits=True)
    assert (h == ho).all()
    assert np.array_equal(lg.view(np.uint64), lo.view(np.uint64))


def test_linear_manhattan_reproduces_manhattan():
    g = np.load(os.path.join(GOLDEN, "manhattan_stp4_c72.npz"))
    with bida.LinearModelBackend("stp4", manhattan_linear_weights(4, 72, 4.0), 72, 0.5) as be:
        h = be.evaluate(g["packed"])
    assert (h == g["h"]).all() and (h == g["manhattan"]).all()


def test_known_answers():
    """test_batch_eval.cpp:153-178 on the device."""
    w = np.zeros((2, 81), np.float32)
    w[1] = 10.0
    w0 = np.zeros((2, 81), np.float32)
    w0[0] = 10.0
    solved = np.array([sum(i << (4 * i) for i in range(9))], np.uint64)
    with bida.LinearModelBackend("stp3", [w], 2, 0.5) as be:
        assert be.evaluate(solved)[0] == 1
    with bida.LinearModelBackend("stp3", [w, w0], 2, 0.5) as be:
        assert be.evaluate(solved)[0] == 0


@pytest.mark.parametrize(
    "domain,E,C,q",
    [(STP2, 1, 3, 0.5), (STP3, 2, 31, 0.5), (STP3, 1, 32, 1.0), (STP4, 1, 33, 0.5), (STP4, 3, 96, 0.4),
     (RC, 1, 1, 0.5), (RC, 2, 64, 0.75), (RC, 1, 100, 0.05), (RC, 1, 256, 0.5)],
)
def test_shapes_vs_oracle(orc, domain, E, C, q):
    rng = np.random.default_rng(C + 7 * E)
    W = rng.uniform(-0.3, 0.3, (E, C, FEATURES[domain])).astype(np.float32)
    packed = bida.random_walks(domain, 1537, 0, 40, seed=C)
    with bida.LinearModelBackend(domain, W, C, q) as be:
        h = be.evaluate(packed)
    assert (h == orc.linear_evaluate(domain, W, q, packed)).all()


def test_empty_and_ragged_batches(orc):
    rng = np.random.default_rng(1)
    W = rng.uniform(-0.1, 0.1, (1, 21, 480)).astype(np.float32)
    packed = bida.random_walks("rc", 300, 0, 30, seed=2)
    want = orc.linear_evaluate(RC, W, 0.5, packed)
    with bida.LinearModelBackend("rc", W, 21, 0.5) as be:
        assert len(be.evaluate(packed[:0])) == 0
        for n in (1, 2, 31, 32, 33, 63, 255, 300):
            assert (be.evaluate(packed[:n]) == want[:n]).all()


def test_batch_composition_independence(orc):
    """test_batch_eval.cpp:209-224: h does not depend on how states are batched."""
    rng = np.random.default_rng(2)
    W = rng.uniform(-0.1, 0.1, (2, 21, 480)).astype(np.float32)
    packed = bida.random_walks("rc", 640, 0, 30, seed=3)
    with bida.LinearModelBackend("rc", W, 21, 0.5) as be:
        full = be.evaluate(packed)
        for B in (1, 7, 64):
            parts = np.concatenate([be.evaluate(packed[i : i + B]) for i in range(0, len(packed), B)])
            assert (parts == full).all()
    assert (full == orc.linear_evaluate(RC, W, 0.5, packed)).all()


def test_non_finite_weights_replay_dense_loop(orc):
    """inf*0 = NaN in the reference's dense dot: rows with non-finite weights."""
    rng = np.random.default_rng(4)
    W = rng.uniform(-0.1, 0.1, (2, 9, 81)).astype(np.float32)
    W[0, 3, 5] = np.inf
    W[0, 4, 7] = -np.inf
    W[1, 0, 0] = np.nan
    packed = bida.random_walks("stp3", 500, 0, 30, seed=5)
    with bida.LinearModelBackend("stp3", W, 9, 0.5) as be:
        h, lg = be.evaluate_logits(packed)
    ho, lo = orc.linear_evaluate(STP3, W, 0.5, packed, want_logits=True)
    assert (h == ho).all()
    assert np.array_equal(lg.view(np.uint64), lo.view(np.uint64))


def test_malformed_state_is_an_error():
    W = np.zeros((1, 2, 480), np.float32)
    bad = np.zeros(3, bida.instances.packed_dtype("rc"))
    bad["hi"][1] = np.uint64(0xFFFFFFFFFFFF)  # edge cubie ids 15: outside F
    with bida.LinearModelBackend("rc", W, 2, 0.5) as be:
        with pytest.raises(ValueError, match="outside"):
            be.evaluate(bad)
        # the handle stays usable afterwards
        good = bida.random_walks("rc", 5, 0, 5, seed=1)
        assert (be.evaluate(good) >= 0).all()


def test_blin1_file_round_trip(tmp_path, orc):
    rng = np.random.default_rng(6)
    W = rng.uniform(-1, 1, (2, 3, 81)).astype(np.float32)
    path = str(tmp_path / "w.blin")
    bida.LinearModelBackend.save("stp3", path, W, 3)
    packed = bida.random_walks("stp3", 20, 30, 30, seed=6)
    with bida.LinearModelBackend.load("stp3", path, 0.5) as a, bida.LinearModelBackend("stp3", W, 3, 0.5) as b:
        assert (a.evaluate(packed) == b.evaluate(packed)).all()
        assert a.info().ensemble == 2 and a.info().classes == 3


def test_large_batch_pipelined_chunks(orc):
    """3.1M states: crosses the 2^20 staging slot three times; checked on a
    strided sample against the oracle and by batch-composition equality."""
    rng = np.random.default_rng(8)
    W = rng.uniform(-0.1, 0.1, (1, 21, 480)).astype(np.float32)
    n = 3 * (1 << 20) + 12345
    packed = bida.random_walks("rc", n, 0, 30, seed=9)
    with bida.LinearModelBackend("rc", W, 21, 0.5) as be:
        h = be.evaluate(packed)
        sample = np.arange(0, n, 997)
        assert (h[sample] == orc.linear_evaluate(RC, W, 0.5, packed[sample])).all()
        tail = be.evaluate(packed[-5000:])
        assert (tail == h[-5000:]).all()


def test_device_resident_path(orc):
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(10)
    W = rng.uniform(-0.1, 0.1, (1, 21, 480)).astype(np.float32)
    packed = bida.random_walks("rc", 10000, 0, 30, seed=11)
    d_in = torch.from_numpy(packed.view(np.uint8).copy()).cuda()
    d_h = torch.empty(len(packed), dtype=torch.int32, device="cuda")
    with bida.LinearModelBackend("rc", W, 21, 0.5) as be:
        be.evaluate_device(d_in, d_h)
        torch.cuda.synchronize()
        be.status()
        assert (d_h.cpu().numpy() == orc.linear_evaluate(RC, W, 0.5, packed)).all()


def test_concurrent_callers_share_a_handle(orc):
    """Agent thread + evaluate_single/evaluate_sync callers (batch_eval.hpp:241,261)."""
    import threading

    rng = np.random.default_rng(12)
    W = rng.uniform(-0.1, 0.1, (1, 21, 480)).astype(np.float32)
    batches = [bida.random_walks("rc", 100 + 50 * i, 0, 30, seed=i) for i in range(8)]
    want = [orc.linear_evaluate(RC, W, 0.5, b) for b in batches]
    errors = []
    with bida.LinearModelBackend("rc", W, 21, 0.5) as be:
        def work(i):
            for _ in range(20):
                if not (be.evaluate(batches[i]) == want[i]).all():
                    errors.append(i)
        th = [threading.Thread(target=work, args=(i,)) for i in range(8)]
        [t.start() for t in th]
        [t.join() for t in th]
    assert not errors


@pytest.mark.parametrize("q", [0.25, 0.5, 0.75, 1.0, 0.3])
def test_exact_ties_take_exact_replay(orc, q):
    """Zero weights: uniform softmax, cum_k = (k+1)/C lands exactly on q -
    the certified float32 readout must defer to the float64 replay."""
    W = np.zeros((1, 4, 480), np.float32)
    packed = bida.random_walks("rc", 200, 0, 20, seed=3)
    with bida.LinearModelBackend("rc", W, 4, q) as be:
        h = be.evaluate(packed)
    assert (h == orc.linear_evaluate(RC, W, q, packed)).all()


@pytest.mark.parametrize("scale,C", [(50.0, 21), (1e-6, 21), (5.0, 200)])
def test_extreme_logit_scales(orc, scale, C):
    rng = np.random.default_rng(int(scale * 7) + C)
    W = rng.uniform(-scale, scale, (2, C, 480)).astype(np.float32)
    packed = bida.random_walks("rc", 1500, 0, 30, seed=C)
    for q in (0.5, 0.999, 1.0, 0.001):
        with bida.LinearModelBackend("rc", W, C, q) as be:
            h = be.evaluate(packed)
        assert (h == orc.linear_evaluate(RC, W, q, packed)).all(), q


def test_concurrent_callers_on_one_handle(orc):
    """The C-ABI handle is re-entrant: 8 host threads hammer one
    handle with small (zero-copy lane) and large (staged slot) batches at
    once; every result is bit-exact against the oracle."""
    import threading

    rng = np.random.default_rng(77)
    W = rng.uniform(-0.1, 0.1, (2, 21, 480)).astype(np.float32)
    batches = [bida.random_walks("rc", n, 0, 30, seed=100 + i)
               for i, n in enumerate([1, 7, 513, 4096, 32768, 40000, 3000, 1 << 16] * 2)]
    want = [orc.linear_evaluate(RC, W, 0.5, b) for b in batches]
    got = [None] * len(batches)
    with bida.LinearModelBackend("rc", W, 21, 0.5) as be:
        def work(t):
            for _ in range(3):
                for i in range(t, len(batches), 8):
                    got[i] = be.evaluate(batches[i])
        ths = [threading.Thread(target=work, args=(t,)) for t in range(8)]
        for th in ths:
            th.start()
        for th in ths:
            th.join()
    for g_, w_ in zip(got, want):
        assert (g_ == w_).all()
