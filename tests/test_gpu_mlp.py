"""GPU parity of the tcgen05 BMLP1 evaluator against the oracle's BMLP1
restatement (oracle/bida_oracle.c), through the C-ABI.  Integer logits are
exact, so the bar is bit-exact logits and h on every state; the certified
float32 readout must agree with the float64 reference sequence everywhere,
including the ties that force its exact replay."""
import numpy as np
import pytest

import paper_2507_11916_b200 as bida
from oracle_lib import RC, STP2, STP3, STP4, Oracle
from paper_2507_11916_b200.models import BMLP1, Layer, make_bmlp1

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def orc():
    return Oracle()


def check(orc, domain, blob, q, packed, E, C):
    with bida.MlpModelBackend(domain, blob, q) as be:
        h, lg = be.evaluate_logits(packed)
        h2 = be.evaluate(packed)
    ho, lo = orc.mlp_evaluate(blob, domain, q, packed, want_logits=True, E=E, Cc=C, threads=8)
    assert np.array_equal(lg.view(np.uint64), lo.view(np.uint64)), "logits differ"
    assert (h == ho).all(), f"{(h != ho).sum()} h flips"
    assert (h2 == ho).all()
    return h


@pytest.mark.parametrize(
    "domain,hidden,C,E,q",
    [
        (RC, [128, 128], 21, 1, 0.5),
        (RC, [128, 128], 21, 2, 0.3),
        (RC, [512, 512], 21, 1, 0.5),
        (RC, [256], 27, 1, 0.9),
        (RC, [64, 96, 128], 40, 3, 0.5),
        (STP4, [256, 256], 72, 1, 0.5),
        (STP4, [128], 64, 2, 1.0),
        (STP3, [64, 64], 32, 1, 0.5),
        (STP2, [32], 7, 1, 0.05),
    ],
)
def test_mlp_matches_oracle(orc, domain, hidden, C, E, q):
    blob = make_bmlp1(domain, hidden=hidden, classes=C, ensemble=E, seed=sum(hidden) + C)
    packed = bida.random_walks(domain, 1000, 0, 40, seed=C)
    h = check(orc, domain, blob, q, packed, E, C)
    if q < 0.99:  # at q = 1 every state correctly reads out the top class
        assert len(np.unique(h)) > 1


def test_ragged_and_empty(orc):
    blob = make_bmlp1("rc", hidden=[128, 128], classes=21, ensemble=1, seed=3)
    packed = bida.random_walks("rc", 700, 0, 30, seed=4)
    want = orc.mlp_evaluate(blob, RC, 0.5, packed, threads=8)
    with bida.MlpModelBackend("rc", blob, 0.5) as be:
        assert len(be.evaluate(packed[:0])) == 0
        for n in (1, 127, 128, 129, 255, 256, 257, 700):
            assert (be.evaluate(packed[:n]) == want[:n]).all(), n


def test_ties_force_exact_replay(orc):
    """All-zero weights: uniform softmax, cum hits q exactly at class C*q-1 —
    undecidable in float32, so every state takes the float64 replay."""
    m = BMLP1(480, 4, [32])
    layers = [Layer(np.zeros((32, 480), np.int8), np.zeros(32, np.int32), 0),
              Layer(np.zeros((4, 32), np.int8), np.zeros(4, np.int32), 0)]
    m.members.append((layers, 1.0))
    blob = m.to_bytes()
    packed = bida.random_walks("rc", 300, 0, 20, seed=1)
    for q in (0.25, 0.5, 0.75, 1.0, 0.3):
        h = check(orc, RC, blob, q, packed, 1, 4)
        assert len(np.unique(h)) == 1


def test_saturated_logits(orc):
    """Huge out_scale: logits ~1e6 -> float32 bound gives up, exact path decides."""
    blob = make_bmlp1("rc", hidden=[64], classes=21, ensemble=1, seed=9, logit_std=5e5)
    packed = bida.random_walks("rc", 400, 0, 30, seed=2)
    check(orc, RC, blob, 0.5, packed, 1, 21)


def test_large_batch_composition(orc):
    blob = make_bmlp1("rc", hidden=[256, 256], classes=21, ensemble=1, seed=11)
    n = (1 << 20) + 333
    packed = bida.random_walks("rc", n, 0, 30, seed=12)
    with bida.MlpModelBackend("rc", blob, 0.5) as be:
        h = be.evaluate(packed)
        sample = np.arange(0, n, 509)
        assert (h[sample] == orc.mlp_evaluate(blob, RC, 0.5, packed[sample], threads=8)).all()
        parts = np.concatenate([be.evaluate(packed[i : i + 77777]) for i in range(0, 400000, 77777)])
        assert (parts == h[: len(parts)]).all()


def test_malformed_state_is_an_error():
    blob = make_bmlp1("rc", hidden=[64], classes=21, ensemble=1, seed=1)
    bad = np.zeros(3, bida.instances.packed_dtype("rc"))
    bad["hi"][1] = np.uint64(0xFFFFFFFFFFFF)
    with bida.MlpModelBackend("rc", blob, 0.5) as be:
        with pytest.raises(ValueError, match="outside"):
            be.evaluate(bad)
        good = bida.random_walks("rc", 5, 0, 5, seed=1)
        assert (be.evaluate(good) >= 0).all()


@pytest.mark.parametrize("hidden", [[64], [600]])
def test_out_of_range_edge_labels(hidden):
    """Every edge slot p and label v: v >= 12 puts the feature index past F (an
    error, rubiks.hpp:155-166 indexing), v <= 11 does not (the kernels' bit test
    on the packed hi word must equal the per-position range check); both the
    fused and the wide schedule."""
    blob = make_bmlp1("rc", hidden=hidden, classes=21, ensemble=1, seed=2)
    base = bida.random_walks("rc", 1, 0, 0, seed=1)
    with bida.MlpModelBackend("rc", blob, 0.5) as be:
        for p in range(12):
            for v in (11, 12, 13, 14, 15):
                st = base.copy()
                hi = int(st["hi"][0]) & ~(0xF << (4 * p))
                st["hi"][0] = np.uint64(hi | (v << (4 * p)))
                if v >= 12:
                    with pytest.raises(ValueError, match="outside"):
                        be.evaluate(st)
                else:
                    assert be.evaluate(st)[0] >= 0


def test_device_resident(orc):
    torch = pytest.importorskip("torch")
    blob = make_bmlp1("rc", hidden=[128, 128], classes=21, ensemble=1, seed=21)
    packed = bida.random_walks("rc", 5000, 0, 30, seed=22)
    d_in = torch.from_numpy(packed.view(np.uint8).copy()).cuda()
    d_h = torch.empty(len(packed), dtype=torch.int32, device="cuda")
    with bida.MlpModelBackend("rc", blob, 0.5) as be:
        be.evaluate_device(d_in, d_h)
        torch.cuda.synchronize()
        be.status()
    assert (d_h.cpu().numpy() == orc.mlp_evaluate(blob, RC, 0.5, packed, threads=8)).all()


def test_bad_models_rejected():
    with pytest.raises(ValueError):
        bida.MlpModelBackend("rc", make_bmlp1("rc", hidden=[4097], classes=21, seed=1), 0.5)  # > 4096
    with pytest.raises(RuntimeError):
        bida.MlpModelBackend("rc", b"BMLP1" + b"\0" * 8, 0.5)
    with pytest.raises(RuntimeError):
        bida.MlpModelBackend("stp4", make_bmlp1("rc", hidden=[64], classes=21, seed=1), 0.5)


@pytest.mark.parametrize("schedule", ["wide", "resident", "pair", "split"])
@pytest.mark.parametrize(
    "hidden,C,E",
    [([128, 128], 21, 1), ([96, 160], 21, 1), ([64, 256, 96], 27, 2), ([256, 64], 40, 1), ([32], 7, 3)],
)
def test_every_schedule_matches_oracle(orc, monkeypatch, schedule, hidden, C, E):
    """The kernel schedules (wide / resident weights / tile ping-pong / N-half
    pipelined split) give identical, oracle-exact results, including odd
    K-chunk splits (96, 160) and layers wider than the previous one.  Three
    CTAs: several tiles each, so both slots of the two-tile schedules run."""
    monkeypatch.setenv("BIDA_MLP_MAX_CTAS", "3")
    monkeypatch.setenv("BIDA_MLP_FORCE_MODE", schedule)
    blob = make_bmlp1("rc", hidden=hidden, classes=C, ensemble=E, seed=len(hidden) * 100 + C)
    packed = bida.random_walks("rc", 777, 0, 30, seed=C + E)
    check(orc, RC, blob, 0.5, packed, E, C)


@pytest.mark.parametrize("multicast", ["0", "1"])
@pytest.mark.parametrize("schedule,hidden", [("pair", [256, 256]), ("split", [512, 512]), ("split", [96, 160])])
def test_cluster_multicast_on_and_off(orc, monkeypatch, multicast, schedule, hidden):
    """Streaming schedules optionally run as CTA pairs sharing weight stages by
    TMA multicast (BIDA_MLP_MULTICAST=1); both paths must agree with the oracle.
    1001 states -> 8 tiles: pairs whose odd CTA gets an empty surplus tile."""
    monkeypatch.setenv("BIDA_MLP_FORCE_MODE", schedule)
    monkeypatch.setenv("BIDA_MLP_MULTICAST", multicast)
    blob = make_bmlp1("rc", hidden=hidden, classes=21, ensemble=1, seed=sum(hidden))
    for n in (1001, 148 * 128 * 2 + 77):
        packed = bida.random_walks("rc", n, 0, 30, seed=n)
        check(orc, RC, blob, 0.5, packed, 1, 21)


@pytest.mark.parametrize(
    "hidden,C,E,q,ctas",
    [([1610, 1610], 21, 1, 0.5, 3), ([600], 27, 2, 0.3, 2), ([1024, 2048, 64], 40, 1, 0.5, 5),
     ([33, 700], 7, 3, 0.9, 1), ([512, 512], 21, 1, 0.5, 148)],
)
@pytest.mark.parametrize("pair", ["1", "0"])
def test_wide_schedule_matches_oracle(orc, monkeypatch, hidden, C, E, q, ctas, pair):
    """Wide hidden layers (the paper's 13.6 MB anchor, H = 1610, and widths that
    are not multiples of the 512-column chunk or of 32): activations round-trip
    through the per-CTA global scratch.  Few CTAs -> many tiles per CTA; an odd
    CTA cap leaves a CTA pair with empty tiles.  pair=1: M = 256 MMAs across a
    CTA pair (cta_group::2), pair=0: one CTA per tile."""
    monkeypatch.setenv("BIDA_MLP_MAX_CTAS", str(ctas))
    monkeypatch.setenv("BIDA_MLP_WIDE_PAIR", pair)
    blob = make_bmlp1("rc", hidden=hidden, classes=C, ensemble=E, seed=sum(hidden) + C)
    packed = bida.random_walks("rc", 128 * 7 + 45 if ctas < 148 else 2000, 0, 30, seed=C)
    h = check(orc, RC, blob, q, packed, E, C)
    assert len(np.unique(h)) > 1
