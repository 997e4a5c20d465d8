"""GPU: PDB-correction readout (north star).  The device
computes Abstraction::rank_state and PdbTable::lookup (pdb.hpp:66-69) inside
the fused readout; checked against PDBs built and looked up by the reference
itself (tests/golden/pdb_*.npz) and the oracle's model h."""
import glob
import os
import struct

import numpy as np
import pytest

import paper_2507_11916_b200 as bida
from oracle_lib import Oracle
from paper_2507_11916_b200.models import make_bmlp1

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
FIX = sorted(glob.glob(os.path.join(GOLDEN, "pdb_*.npz")))
FEAT = {3: 81, 4: 256, 100: 480}


@pytest.fixture(scope="module")
def orc():
    return Oracle()


def bpdb1_bytes(domain, pattern, entries):
    """PdbTable::save layout (pdb.hpp:78-96)."""
    tag, board = (b"R", 0) if domain == 100 else (b"S", domain * domain)
    return (b"BPDB1" + tag + bytes([board, len(pattern)]) + bytes(pattern) + struct.pack("<Q", len(entries))
            + bytes(entries))


@pytest.mark.parametrize("path", FIX)
@pytest.mark.parametrize("kind", ["linear", "mlp"])
def test_pdb_min_and_replace(orc, path, kind):
    g = np.load(path)
    d = int(g["domain"])
    packed, pat, ent, h_pdb = g["packed"], g["pattern"], g["entries"], g["h"]
    if kind == "linear":
        W = np.random.default_rng(d).uniform(-0.1, 0.1, (1, 24, FEAT[d])).astype(np.float32)
        be = bida.LinearModelBackend(d, W, 24, 0.5)
        h_model = orc.linear_evaluate(d, W, 0.5, packed)
    else:
        blob = make_bmlp1(d, hidden=[64, 64], classes=24, ensemble=1, seed=d)
        be = bida.MlpModelBackend(d, blob, 0.5)
        h_model = orc.mlp_evaluate(blob, d, 0.5, packed, threads=8)
    with be:
        assert (be.evaluate(packed) == h_model).all()
        be.attach_pdb(pat, ent, mode="min")
        assert (be.evaluate(packed) == np.minimum(h_model, h_pdb)).all()
        be.attach_pdb(pat, ent, mode="replace")
        assert (be.evaluate(packed) == h_pdb).all()
        be.attach_pdb(None, None, mode="off")
        assert (be.evaluate(packed) == h_model).all()


def test_pdb_from_bpdb1_file_and_errors(tmp_path):
    g = np.load(os.path.join(GOLDEN, "pdb_rc_c4.npz"))
    f = tmp_path / "c4.pdb"
    f.write_bytes(bpdb1_bytes(100, list(g["pattern"]), g["entries"]))
    blob = make_bmlp1("rc", hidden=[64], classes=21, ensemble=1, seed=3)
    with bida.MlpModelBackend("rc", blob, 0.5) as be:
        be.attach_pdb(None, path=str(f), mode="replace")
        assert (be.evaluate(g["packed"]) == g["h"]).all()
        with pytest.raises(ValueError, match="corner labels"):
            be.attach_pdb([0, 9], g["entries"], mode="min")
        with pytest.raises(RuntimeError, match="entry count"):
            be.attach_pdb([0, 1, 2], g["entries"], mode="min")
        bad = tmp_path / "stp.pdb"
        bad.write_bytes(bpdb1_bytes(3, [1, 2], np.zeros(72, np.uint8)))
        with pytest.raises(RuntimeError, match="domain mismatch"):
            be.attach_pdb(None, path=str(bad), mode="min")


def test_pdb_large_batch_and_device_path():
    torch = pytest.importorskip("torch")
    g = np.load(os.path.join(GOLDEN, "pdb_rc_c4.npz"))
    packed = bida.random_walks("rc", 300000, 0, 30, seed=9)
    orc = Oracle()
    h_pdb = orc.pdb_lookup(100, g["pattern"], g["entries"], packed)
    blob = make_bmlp1("rc", hidden=[128, 128], classes=21, ensemble=1, seed=4)
    with bida.MlpModelBackend("rc", blob, 0.5) as be:
        be.attach_pdb(g["pattern"], g["entries"], mode="replace")
        assert (be.evaluate(packed) == h_pdb).all()
        d_in = torch.from_numpy(packed.view(np.uint8).copy()).cuda()
        d_h = torch.empty(len(packed), dtype=torch.int32, device="cuda")
        be.evaluate_device(d_in, d_h)
        torch.cuda.synchronize()
        be.status()
        assert (d_h.cpu().numpy() == h_pdb).all()
