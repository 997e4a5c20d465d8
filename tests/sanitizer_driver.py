"""Small driver for compute-sanitizer runs (SURVEY §5 race detection; VERDICT
r1 next #8): one launch of every kernel family on a few tiles -- the four MLP
schedules (resident, pair, split, wide, forced through BIDA_MLP_FORCE_MODE in
child processes), the thread- and warp-per-state linear kernels, the PDB
readout and the GPU PDB build -- each checked against the oracle.  Not a
pytest test; run as

    compute-sanitizer --tool memcheck python tests/sanitizer_driver.py
"""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def one(kind):
    import paper_2507_11916_b200 as bida
    from oracle_lib import RC, Oracle
    from paper_2507_11916_b200.backend import pdb_build
    from paper_2507_11916_b200.models import make_bmlp1

    orc = Oracle()
    packed = bida.random_walks("rc", 700, 0, 30, seed=3)
    if kind.startswith("mlp"):
        hidden = [512, 512] if kind in ("mlp_wide", "mlp_split") else [128, 128]
        blob = make_bmlp1("rc", hidden=hidden, classes=21, ensemble=2, seed=5)
        with bida.MlpModelBackend("rc", blob, 0.5) as be:
            h = be.evaluate(packed)
        want = orc.mlp_evaluate(blob, RC, 0.5, packed)
    elif kind == "linear_thread":
        W = np.random.default_rng(1).uniform(-0.1, 0.1, (2, 21, 480)).astype(np.float32)
        with bida.LinearModelBackend("rc", W, 21, 0.5) as be:
            be.attach_pdb([0, 1, 2, 3], mode="min")  # PDB build + fused readout
            h = be.evaluate(packed)
        ent = pdb_build("rc", [0, 1, 2, 3])
        want = np.minimum(orc.linear_evaluate(RC, W, 0.5, packed), orc.pdb_lookup(RC, [0, 1, 2, 3], ent, packed))
    elif kind == "linear_warp":
        W = np.random.default_rng(2).uniform(-0.1, 0.1, (1, 100, 480)).astype(np.float32)
        with bida.LinearModelBackend("rc", W, 100, 0.5) as be:
            h = be.evaluate(packed)
        want = orc.linear_evaluate(RC, W, 0.5, packed)
    else:
        raise SystemExit(f"unknown kind {kind}")
    bad = int((h != want).sum())
    print(f"{kind}: {len(h)} states, {bad} differ from the oracle", flush=True)
    return bad


if __name__ == "__main__":
    if len(sys.argv) > 1:
        sys.exit(1 if one(sys.argv[1]) else 0)
    rc = 0
    for kind, mode in [("mlp_resident", "resident"), ("mlp_pair", "pair"), ("mlp_split", "split"),
                       ("mlp_wide", "wide"), ("linear_thread", ""), ("linear_warp", "")]:
        env = {**os.environ, "BIDA_MLP_MAX_CTAS": "2"}
        if mode:
            env["BIDA_MLP_FORCE_MODE"] = mode
        rc |= subprocess.run([sys.executable, __file__, kind], env=env).returncode
    sys.exit(rc)
