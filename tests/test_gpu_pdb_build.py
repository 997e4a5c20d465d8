"""GPU breadth-first PDB construction (bida_gpu_pdb_build; SURVEY §8(f) row 3,
pdb.hpp:30-64) against tables built by the reference itself: byte-identical
entries for small patterns (oracle/_ref PdbTable<D>::build), and the sha256 of
the reference's own BPDB1 files for the 5- to 8-corner Rubik's tables
(tests/golden/pdb_rc_digests.json, make_golden_pdb_sha.py)."""
from __future__ import annotations

import hashlib
import json
import os
import time

import numpy as np
import pytest

import paper_2507_11916_b200 as bida
from oracle_lib import RC, STP3, STP4, RefLib
from paper_2507_11916_b200.backend import pdb_build, pdb_build_save

pytestmark = pytest.mark.gpu

DIGESTS = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "pdb_rc_digests.json")))


def record(**kw):
    out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out")
    if os.path.isdir(out):
        with open(os.path.join(out, "pdb_build.jsonl"), "a") as f:
            f.write(json.dumps(kw) + "\n")


@pytest.mark.parametrize("domain,pattern", [
    (RC, [0]), (RC, [0, 1, 2, 3]), (RC, [7, 2, 5]), (RC, [3, 0, 6, 1, 4]),
    (STP3, [1, 2, 3]), (STP3, [0, 1, 2, 3, 4]), (STP3, [5, 0, 8, 1]), (STP3, [1, 2, 3, 4, 5, 6, 7, 8]),
    (STP4, [1, 2, 3, 4]), (STP4, [0, 1, 2, 3, 4]), (STP4, [15, 11, 14, 7]),
])
def test_matches_reference_build(domain, pattern):
    want = RefLib().pdb_build(domain, pattern)
    got = pdb_build(domain, pattern)
    assert got.shape == want.shape
    assert np.array_equal(got, want), f"{int((got != want).sum())} entries differ"


@pytest.mark.parametrize("corners", [5, 6, 7, 8])
def test_rubiks_corner_tables_match_reference_digest(corners, tmp_path):
    d = DIGESTS[f"rc_c{corners}"]
    path = str(tmp_path / f"rc_c{corners}.pdb")
    t0 = time.time()
    pdb_build_save("rc", list(range(corners)), path)
    secs = time.time() - t0
    data = open(path, "rb").read()
    os.unlink(path)
    ent = np.frombuffer(data, np.uint8, offset=8 + corners + 8)
    hist = {str(k): int(v) for k, v in enumerate(np.bincount(ent, minlength=256)) if v}
    record(test="rc_corner_pdb", corners=corners, entries=len(ent), gpu_build_save_s=secs,
           reference_build_s=d["reference_build_seconds"])
    assert hist == d["depth_histogram"]
    assert len(data) == d["file_bytes"]
    assert hashlib.sha256(data).hexdigest() == d["sha256"]


def test_reference_error_messages():
    with pytest.raises(RuntimeError, match="PDB abstract space needs 518918400 entries, cap is 268435456"):
        pdb_build("stp4", [1, 2, 3, 4, 5, 6, 7, 8])
    with pytest.raises(ValueError, match="only corner labels"):
        pdb_build("rc", [8])
    with pytest.raises(ValueError, match="repeated"):
        pdb_build("stp3", [1, 1])


def test_attach_built_equals_attach_entries():
    rng = np.random.default_rng(3)
    W = rng.uniform(-0.1, 0.1, (1, 21, 480)).astype(np.float32)
    packed = bida.random_walks("rc", 20000, 0, 30, seed=4)
    ent = pdb_build("rc", [0, 1, 2, 3, 4])
    with bida.LinearModelBackend("rc", W, 21, 0.5) as a, bida.LinearModelBackend("rc", W, 21, 0.5) as b:
        a.attach_pdb([0, 1, 2, 3, 4], ent, mode="replace")
        b.attach_pdb([0, 1, 2, 3, 4], mode="replace")  # built on the device
        ha, hb = a.evaluate(packed), b.evaluate(packed)
    assert (ha == hb).all()
    assert (ha == RefLib().pdb_lookup_file(RC, _save(ent, [0, 1, 2, 3, 4]), packed)).all()


def _save(ent, pattern, path="/tmp/_bida_test_c5.pdb"):
    with open(path, "wb") as f:
        f.write(b"BPDB1R\x00" + bytes([len(pattern)]) + bytes(pattern) + len(ent).to_bytes(8, "little"))
        f.write(ent.tobytes())
    return path
