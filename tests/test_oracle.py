"""CPU: the oracle restatement is pinned against the reference itself
(oracle/_ref) and against the committed golden vectors, and the reference's
own known-answer tests for this path are replayed on both."""
import glob
import os

import numpy as np
import pytest

from oracle_lib import FEATURES, RC, REF_SO, STP2, STP3, STP4, Oracle, RefLib, manhattan_linear_weights

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
HAVE_REF = os.path.exists(REF_SO) or os.path.isdir("/root/reference/proj/include")
needs_ref = pytest.mark.skipif(not HAVE_REF, reason="oracle/_ref not built")


@pytest.fixture(scope="module")
def orc():
    return Oracle()


@pytest.fixture(scope="module")
def ref():
    return RefLib()


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLDEN, "linear_*.npz"))))
def test_oracle_matches_golden(orc, path):
    g = np.load(path)
    h = orc.linear_evaluate(int(g["domain"]), g["W"], float(g["q"]), g["packed"])
    assert (h == g["h"]).all()


def test_oracle_linear_manhattan_golden(orc):
    g = np.load(os.path.join(GOLDEN, "manhattan_stp4_c72.npz"))
    W = manhattan_linear_weights(4, 72, 4.0)
    h = orc.linear_evaluate(STP4, W, 0.5, g["packed"])
    assert (h == g["h"]).all()
    assert (h == g["manhattan"]).all()
    assert (orc.manhattan(STP4, g["packed"]) == g["manhattan"]).all()


@needs_ref
@pytest.mark.parametrize("domain", [STP2, STP3, STP4, RC])
def test_encode_matches_reference(orc, ref, domain):
    packed = ref.random_walks(domain, 400, 0, 50, 9)
    assert (ref.repack(domain, packed) == packed).all()
    xo, xr = orc.encode(domain, packed), ref.encode(domain, packed)
    assert (xo == xr).all()
    # injective one-hot with the domain's number of ones (test_state_space.cpp:225-241)
    assert (xo.sum(1) == {STP2: 4, STP3: 9, STP4: 16, RC: 20}[domain]).all()
    for i in range(0, 400, 37):
        idx = orc.active_indices(domain, packed[i : i + 1])
        assert (np.diff(idx) > 0).all()
        assert (np.flatnonzero(xo[i]) == idx).all()


@needs_ref
@pytest.mark.parametrize(
    "domain,E,C,q,scale",
    [(STP2, 1, 7, 0.5, 1.0), (STP3, 3, 32, 0.7, 0.3), (STP4, 2, 64, 0.25, 0.1), (RC, 2, 21, 0.5, 0.1),
     (RC, 1, 1, 1.0, 1.0), (RC, 1, 33, 1.0, 3.0), (RC, 3, 5, 0.01, 0.5)],
)
def test_linear_matches_reference(orc, ref, domain, E, C, q, scale):
    rng = np.random.default_rng(E * 1000 + C)
    packed = ref.random_walks(domain, 600, 0, 40, C)
    W = rng.uniform(-scale, scale, (E, C, FEATURES[domain])).astype(np.float32)
    assert (orc.linear_evaluate(domain, W, q, packed) == ref.linear_evaluate(domain, W, q, packed)).all()


@needs_ref
def test_multithreaded_reference_equals_single(ref):
    rng = np.random.default_rng(3)
    packed = ref.random_walks(RC, 1000, 0, 30, 3)
    W = rng.uniform(-0.1, 0.1, (1, 21, 480)).astype(np.float32)
    assert (ref.linear_evaluate(RC, W, 0.5, packed, threads=4) == ref.linear_evaluate(RC, W, 0.5, packed)).all()


@needs_ref
def test_blin1_round_trip_through_reference(orc, ref, tmp_path):
    """test_batch_eval.cpp:180-207, with the file written by the reference."""
    rng = np.random.default_rng(5)
    W = rng.uniform(-1, 1, (2, 3, 81)).astype(np.float32)
    path = str(tmp_path / "w.blin")
    ref.blin1_save(STP3, path, W)
    packed = ref.random_walks(STP3, 20, 30, 30, 5)
    a = ref.blin1_load_evaluate(STP3, path, 0.5, packed)
    b = ref.linear_evaluate(STP3, W, 0.5, packed)
    assert (a == b).all()
    assert (orc.linear_evaluate(STP3, W, 0.5, packed) == a).all()
    # the package's BLIN1 writer produces the same bytes as the reference's
    from paper_2507_11916_b200.backend import blin1_bytes

    with open(path, "rb") as f:
        assert f.read() == blin1_bytes(STP3, W, 3)


def test_linear_known_answers(orc):
    """test_batch_eval.cpp:153-178: class-1 row of 10s -> 1; ensemble min -> 0."""
    fl = 81
    w = np.zeros((2, fl), np.float32)
    w[1, :] = 10.0
    w0 = np.zeros((2, fl), np.float32)
    w0[0, :] = 10.0
    solved = np.array([sum(i << (4 * i) for i in range(9))], np.uint64)
    assert orc.linear_evaluate(STP3, w[None], 0.5, solved)[0] == 1
    assert orc.linear_evaluate(STP3, np.stack([w, w0]), 0.5, solved)[0] == 0


@pytest.mark.parametrize("impl", ["oracle", "reference"])
def test_quantile_known_answers(orc, impl):
    """test_heuristics.cpp:262-285."""
    if impl == "reference":
        if not HAVE_REF:
            pytest.skip("oracle/_ref not built")
        lib = RefLib()
    else:
        lib = orc
    d = [0.2, 0.4, 0.4]
    assert lib.quantile_class(d, 0.5) == 1
    assert lib.quantile_class(d, 1.0) == 2
    assert lib.quantile_class(d, 0.1) == 0
    for q in (0.01, 0.5, 1.0):
        assert lib.quantile_class([0.0, 0.0, 0.0, 1.0], q) == 3
    prev = 0
    for q in np.arange(0.05, 1.0001, 0.05):
        c = lib.quantile_class([0.1, 0.2, 0.3, 0.4], float(q))
        assert c >= prev
        prev = c
    for bad_q in (0.0, 1.1):
        with pytest.raises(ValueError):
            lib.quantile_class(d, bad_q)
    with pytest.raises(ValueError):
        lib.quantile_class([0.5, 0.1], 0.5)


@needs_ref
def test_ensemble_min_known_answers(ref):
    """test_heuristics.cpp:287-293."""
    assert ref.ensemble_min([3, 5, 4]) == 3
    assert ref.ensemble_min([7]) == 7
    with pytest.raises(ValueError):
        ref.ensemble_min([])


@needs_ref
def test_golden_fixtures_reproduce_from_reference(ref):
    """The committed fixtures are what the reference produces (regenerable)."""
    g = np.load(os.path.join(GOLDEN, "linear_rc_e1_c21.npz"))
    packed = ref.random_walks(RC, len(g["packed"]), 0, 30, 1000 + 104)
    assert (packed == g["packed"]).all()
    assert (ref.linear_evaluate(RC, g["W"], float(g["q"]), packed) == g["h"]).all()


def test_package_walks_are_valid_states(orc):
    import paper_2507_11916_b200 as bida

    for d in (STP2, STP3, STP4, RC):
        packed = bida.random_walks(d, 3000, 0, 40, 1)
        x = orc.encode(d, packed)
        assert (x.sum(1) == {STP2: 4, STP3: 9, STP4: 16, RC: 20}[d]).all()
        if HAVE_REF:
            assert (RefLib().repack(d, packed) == packed).all()


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLDEN, "pdb_*.npz"))))
def test_pdb_rank_lookup_matches_reference_golden(orc, path):
    """orc_pdb_rank/lookup restate Abstraction::rank_state + PdbTable::lookup."""
    g = np.load(path)
    h = orc.pdb_lookup(int(g["domain"]), g["pattern"], g["entries"], g["packed"])
    assert (h == g["h"]).all()
