"""Synthetic-input generator on the device (bida_gpu_random_walks): every
state is a reachable, validly packed scramble with the requested walk length
distribution, and the generator is deterministic per seed."""
import numpy as np
import pytest

import paper_2507_11916_b200 as bida
from oracle_lib import RC, STP4, Oracle

pytestmark = pytest.mark.gpu


def rc_unpack(p):
    lo, hi = p["lo"].astype(np.uint64), p["hi"].astype(np.uint64)
    cp = np.stack([(lo >> np.uint64(3 * i)) & np.uint64(7) for i in range(8)], 1).astype(int)
    co = np.stack([(lo >> np.uint64(24 + 2 * i)) & np.uint64(3) for i in range(8)], 1).astype(int)
    eo = np.stack([(lo >> np.uint64(40 + i)) & np.uint64(1) for i in range(12)], 1).astype(int)
    ep = np.stack([(hi >> np.uint64(4 * i)) & np.uint64(15) for i in range(12)], 1).astype(int)
    return cp, co, ep, eo


def parity(perm):
    inv = np.zeros(len(perm), int)
    for i in range(perm.shape[1]):
        for j in range(i + 1, perm.shape[1]):
            inv += perm[:, i] > perm[:, j]
    return inv % 2


def test_rc_walks_are_valid_cubes():
    n = 200_000
    p = bida.random_walks_fast("rc", n, 0, 30, seed=7)
    cp, co, ep, eo = rc_unpack(p)
    assert (np.sort(cp, 1) == np.arange(8)).all() and (np.sort(ep, 1) == np.arange(12)).all()
    assert (co.max() <= 2) and (co.sum(1) % 3 == 0).all() and (eo.sum(1) % 2 == 0).all()
    assert (parity(cp) == parity(ep)).all()                      # RubiksCube::valid (rubiks.hpp)
    solved = (cp == np.arange(8)).all(1) & (ep == np.arange(12)).all(1) & (co == 0).all(1) & (eo == 0).all(1)
    assert solved[::31].all()                                   # length-0 walks (i % 31 == 0)
    assert solved.mean() < 0.05
    q = bida.random_walks_fast("rc", n, 0, 30, seed=7)
    assert (q == p).all()                                       # deterministic per seed
    assert not (bida.random_walks_fast("rc", n, 0, 30, seed=8) == p).all()


def test_stp_walks_are_valid_puzzles_and_evaluate_like_the_oracle():
    n = 100_000
    p = bida.random_walks_fast("stp4", n, 0, 60, seed=3)
    v = p.astype(np.uint64)
    tiles = np.stack([(v >> np.uint64(4 * c)) & np.uint64(15) for c in range(16)], 1).astype(int)
    assert (np.sort(tiles, 1) == np.arange(16)).all()
    # solvability: permutation parity + blank row distance parity stays even for 4x4
    blank = np.argmax(tiles == 0, 1)
    assert ((parity(tiles) + blank // 4 + blank % 4) % 2 == 0).all()
    W = np.random.default_rng(1).uniform(-0.1, 0.1, (1, 64, 256)).astype(np.float32)
    with bida.LinearModelBackend("stp4", W, 64, 0.5) as be:
        h = be.evaluate(p)
    assert (h == Oracle().linear_evaluate(STP4, W, 0.5, p)).all()
    r = bida.random_walks_fast("rc", 50_000, 14, 16, seed=2)
    with bida.LinearModelBackend("rc", np.zeros((1, 2, 480), np.float32) + 0.01, 2, 0.5) as be:
        assert (be.evaluate(r) == Oracle().linear_evaluate(RC, np.zeros((1, 2, 480), np.float32) + 0.01, 0.5, r)).all()
