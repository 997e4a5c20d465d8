"""Regenerates the golden fixtures in tests/golden/ FROM THE REFERENCE ITSELF.

Runs in the build container only (needs /root/reference): the reference's
headers are compiled unchanged into oracle/_ref/libbida_ref.so, and every h
value stored here is produced by bida::LinearModelBackend<D>::evaluate
(batch_eval.hpp:98-105) on states produced by bida::random_walk_instance
(instance.hpp:36-57) / load_instances (instance.hpp:165-171).  The GPU box
reads only the committed .npz files.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle_lib import RC, STP3, STP4, RefLib, manhattan_linear_weights  # noqa: E402

DATA = "/root/reference/proj/data"


def weights(seed, E, C, F, lo=-0.1, hi=0.1):
    rng = np.random.default_rng(seed)
    return rng.uniform(lo, hi, (E, C, F)).astype(np.float32)


def main() -> None:
    ref = RefLib()
    cases = [
        # name, domain, E, C, q, n, walk lengths, weight seed, weight range
        ("linear_stp3_e2_c32", STP3, 2, 32, 0.5, 3000, (0, 40), 101, 0.1),
        ("linear_stp4_e1_c64", STP4, 1, 64, 0.5, 3000, (0, 60), 102, 0.1),
        ("linear_stp4_e2_c72_q03", STP4, 2, 72, 0.3, 2000, (0, 60), 103, 0.5),
        ("linear_rc_e1_c21", RC, 1, 21, 0.5, 3000, (0, 30), 104, 0.1),
        ("linear_rc_e4_c21_q02", RC, 4, 21, 0.2, 2000, (0, 30), 105, 1.0),
        ("linear_rc_e1_c40_q09", RC, 1, 40, 0.9, 2000, (0, 30), 106, 2.0),
    ]
    for name, d, E, C, q, n, (lmin, lmax), seed, rng_w in cases:
        packed = ref.random_walks(d, n, lmin, lmax, 1000 + seed)
        W = weights(seed, E, C, {STP3: 81, STP4: 256, RC: 480}[d], -rng_w, rng_w)
        h = ref.linear_evaluate(d, W, q, packed)
        np.savez_compressed(os.path.join(HERE, name + ".npz"), domain=d, packed=packed, W=W, q=q, h=h)
        print(name, np.bincount(h))

    # Linear-Manhattan weights reproduce ManhattanHeuristic<N>:
    # Korf's 10 instances (proj/data/korf10.txt) plus reference walks.
    korf = ref.load_instances(STP4, os.path.join(DATA, "korf10.txt"))
    walks = ref.random_walks(STP4, 2000, 0, 80, 77)
    packed = np.concatenate([korf, walks])
    W = manhattan_linear_weights(4, 72, 4.0)
    h = ref.linear_evaluate(STP4, W, 0.5, packed)
    md = ref.manhattan(STP4, packed)
    assert (h == md).all(), "linear-Manhattan weights must reproduce Manhattan"
    np.savez_compressed(os.path.join(HERE, "manhattan_stp4_c72.npz"), domain=STP4, packed=packed, q=0.5,
                        h=h, manhattan=md, n_korf=len(korf))
    print("manhattan_stp4", len(packed))

    # Pattern databases built by the reference (PdbTable<D>::build, pdb.hpp:30-64)
    # and its lookups (pdb.hpp:66-69) on reference walks.
    for name, d, pat, lmax in [("pdb_rc_c4", RC, [0, 1, 2, 3], 30), ("pdb_stp3_p5", STP3, [1, 2, 3, 4, 5], 40),
                               ("pdb_stp4_p4", STP4, [1, 2, 3, 4], 60)]:
        entries = ref.pdb_build(d, pat)
        packed = ref.random_walks(d, 2000, 0, lmax, 4242)
        path = "/tmp/_golden.pdb"
        ref.pdb_build_save(d, pat, path)
        h = ref.pdb_lookup_file(d, path, packed)
        np.savez_compressed(os.path.join(HERE, name + ".npz"), domain=d, pattern=np.array(pat, np.uint8),
                            entries=entries, packed=packed, h=h)
        print(name, len(entries), np.bincount(h))

    stp8 = ref.load_instances(STP3, os.path.join(DATA, "stp8_100.txt"))
    rc50 = ref.load_instances(RC, os.path.join(DATA, "rc50.txt"))
    np.savez_compressed(os.path.join(HERE, "instances.npz"), korf10=korf, stp8_100=stp8, rc50=rc50)
    print("instances", len(korf), len(stp8), len(rc50))


if __name__ == "__main__":
    main()
