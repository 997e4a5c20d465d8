"""Domain constants and synthetic packed-state generators (numpy, vectorised).

The evaluator consumes states packed exactly like the reference packs them:
  * TilePuzzle<N>::pack  (stp.hpp:121-126): u64, tiles[cell] in bits 4*cell.
  * RubiksCube::pack     (rubiks.hpp:126-137): lo = cp (3 bits each) |
    co (2 bits each) << 24 | eo (1 bit each) << 40; hi = ep (4 bits each).

`random_walks` produces seeded random-walk scrambles (the synthetic workload of
SURVEY.md §8(d)): each step picks uniformly among the legal actions minus the
one that retracts the previous step, as random_walk_instance does
(instance.hpp:36-57).  The RNG is numpy's, not mt19937_64, so the states are
not the reference's walks — parity tests that need the reference's own walks
get them from oracle/_ref.
"""
from __future__ import annotations

import numpy as np

STP2, STP3, STP4, RC = 2, 3, 4, 100
DOMAIN_IDS = {"stp2": STP2, "stp3": STP3, "stp4": STP4, "rc": RC}
FEATURES = {STP2: 16, STP3: 81, STP4: 256, RC: 480}
PACKED_BYTES = {STP2: 8, STP3: 8, STP4: 8, RC: 16}
ACTIVE = {STP2: 4, STP3: 9, STP4: 16, RC: 20}


def domain_id(domain) -> int:
    if isinstance(domain, str):
        try:
            return DOMAIN_IDS[domain.lower()]
        except KeyError:
            raise ValueError(f"unknown domain {domain!r}") from None
    d = int(domain)
    if d not in FEATURES:
        raise ValueError(f"unknown domain {domain!r}")
    return d


def packed_dtype(domain) -> np.dtype:
    d = domain_id(domain)
    return np.dtype("<u8") if d != RC else np.dtype([("lo", "<u8"), ("hi", "<u8")])


# ---------------------------------------------------------------- Rubik's
# Clockwise quarter-turn tables of rubiks.hpp:340-364 (cf/ef: position whose
# cubie moves to position i; co/eo: twist added on arrival), U D L R F B.
_Q = [
    ([3, 0, 1, 2, 4, 5, 6, 7], [0] * 8, [3, 0, 1, 2, 4, 5, 6, 7, 8, 9, 10, 11], [0] * 12),
    ([0, 1, 2, 3, 5, 6, 7, 4], [0] * 8, [0, 1, 2, 3, 5, 6, 7, 4, 8, 9, 10, 11], [0] * 12),
    ([0, 2, 6, 3, 4, 1, 5, 7], [0, 1, 2, 0, 0, 2, 1, 0], [0, 1, 10, 3, 4, 5, 9, 7, 8, 2, 6, 11], [0] * 12),
    ([4, 1, 2, 0, 7, 5, 6, 3], [2, 0, 0, 1, 1, 0, 0, 2], [8, 1, 2, 3, 11, 5, 6, 7, 4, 9, 10, 0], [0] * 12),
    ([1, 5, 2, 3, 0, 4, 6, 7], [1, 2, 0, 0, 2, 1, 0, 0], [0, 9, 2, 3, 4, 8, 6, 7, 1, 5, 10, 11],
     [0, 1, 0, 0, 0, 1, 0, 0, 1, 1, 0, 0]),
    ([0, 1, 3, 7, 4, 5, 2, 6], [0, 0, 1, 2, 0, 0, 2, 1], [0, 1, 2, 11, 4, 5, 6, 10, 8, 9, 3, 7],
     [0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 1, 1]),
]


def _compose(a, b):
    """Move table of applying a then b (rubiks.hpp:324-338)."""
    acf, aco, aef, aeo = a
    bcf, bco, bef, beo = b
    cf = [acf[bcf[i]] for i in range(8)]
    co = [(aco[bcf[i]] + bco[i]) % 3 for i in range(8)]
    ef = [aef[bef[i]] for i in range(12)]
    eo = [(aeo[bef[i]] + beo[i]) % 2 for i in range(12)]
    return cf, co, ef, eo


def _rc_tables():
    allt = []
    for f in range(6):
        q1 = _Q[f]
        q2 = _compose(q1, q1)
        q3 = _compose(q2, q1)
        allt += [q1, q2, q3]
    cf = np.array([t[0] for t in allt], np.int64)
    co = np.array([t[1] for t in allt], np.int64)
    ef = np.array([t[2] for t in allt], np.int64)
    eo = np.array([t[3] for t in allt], np.int64)
    return cf, co, ef, eo


_RC = _rc_tables()


def rc_apply(cp, co, ep, eo, a):
    """Vectorised RubiksCube::apply (rubiks.hpp:75-91); a is an action per row."""
    cf, cot, ef, eot = _RC
    rows = np.arange(len(a))[:, None]
    src_c = cf[a]
    src_e = ef[a]
    ncp = cp[rows, src_c]
    nco = (co[rows, src_c] + cot[a]) % 3
    nep = ep[rows, src_e]
    neo = (eo[rows, src_e] + eot[a]) % 2
    return ncp, nco, nep, neo


def rc_pack(cp, co, ep, eo) -> np.ndarray:
    n = len(cp)
    out = np.zeros(n, packed_dtype(RC))
    lo = np.zeros(n, np.uint64)
    hi = np.zeros(n, np.uint64)
    for i in range(8):
        lo |= cp[:, i].astype(np.uint64) << np.uint64(3 * i)
        lo |= co[:, i].astype(np.uint64) << np.uint64(24 + 2 * i)
    for i in range(12):
        lo |= eo[:, i].astype(np.uint64) << np.uint64(40 + i)
        hi |= ep[:, i].astype(np.uint64) << np.uint64(4 * i)
    out["lo"] = lo
    out["hi"] = hi
    return out


def stp_pack(tiles: np.ndarray) -> np.ndarray:
    v = np.zeros(len(tiles), np.uint64)
    for c in range(tiles.shape[1]):
        v |= tiles[:, c].astype(np.uint64) << np.uint64(4 * c)
    return v


def random_walks(domain, n: int, len_min: int = 0, len_max: int = 30, seed: int = 0) -> np.ndarray:
    """n packed states, state i a non-retracting random walk of length
    len_min + i % (len_max - len_min + 1) from the solved state."""
    d = domain_id(domain)
    rng = np.random.default_rng(seed)
    lengths = len_min + (np.arange(n) % (len_max - len_min + 1))
    steps = int(lengths.max()) if n else 0
    if d == RC:
        cp = np.tile(np.arange(8), (n, 1))
        co = np.zeros((n, 8), np.int64)
        ep = np.tile(np.arange(12), (n, 1))
        eo = np.zeros((n, 12), np.int64)
        last_face = np.full(n, -1)
        for s in range(steps):
            live = lengths > s
            # 15 actions: the 5 faces other than the last one, 3 turns each
            r = rng.integers(0, 15 + 3 * (last_face < 0), size=n)
            face = r // 3
            face = np.where((last_face >= 0) & (face >= last_face), face + 1, face)
            a = face * 3 + r % 3
            ncp, nco, nep, neo = rc_apply(cp, co, ep, eo, a)
            m = live[:, None]
            cp, co = np.where(m, ncp, cp), np.where(m, nco, co)
            ep, eo = np.where(m, nep, ep), np.where(m, neo, eo)
            last_face = np.where(live, face, last_face)
        return rc_pack(cp, co, ep, eo)
    N = d
    K = N * N
    tiles = np.tile(np.arange(K), (n, 1))
    blank = np.zeros(n, np.int64)
    last = np.full(n, -1)
    rows = np.arange(n)
    # actions: up(-N), down(+N), left(-1), right(+1); inverse = a ^ 1 (stp.hpp:79)
    deltas = np.array([-N, N, -1, 1])
    for s in range(steps):
        live = lengths > s
        r, c = blank // N, blank % N
        legal = np.stack([r > 0, r < N - 1, c > 0, c < N - 1], 1)
        legal[rows[last >= 0], (last[last >= 0] ^ 1)] = False
        cnt = legal.sum(1)
        pick = (rng.random(n) * cnt).astype(np.int64)
        order = np.cumsum(legal, 1) - 1
        a = np.argmax(legal & (order == pick[:, None]), 1)
        target = blank + deltas[a]
        nt = tiles.copy()
        nt[rows, blank] = tiles[rows, target]
        nt[rows, target] = 0
        tiles = np.where(live[:, None], nt, tiles)
        blank = np.where(live, target, blank)
        last = np.where(live, a, last)
    return stp_pack(tiles)
