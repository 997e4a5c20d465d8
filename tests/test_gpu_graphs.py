"""Zero-copy lanes replay a per-lane CUDA graph (bida_gpu.cu lane_launch):
every small batch is one graph launch whose kernel-node parameters (n, grid,
shared memory, PDB) are rewritten per call.  Results must stay bit-exact
across batch-size changes on the same lane, and BIDA_GPU_GRAPHS=0 must give
the same h through plain launches."""
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_2507_11916_b200 as bida
from oracle_lib import RC, Oracle
from paper_2507_11916_b200.models import make_bmlp1

pytestmark = pytest.mark.gpu
SIZES = [1, 300, 4096, 7, 32768, 129, 4097, 2]


def backend(model):
    if model == "linear":
        W = np.random.default_rng(11).uniform(-0.1, 0.1, (2, 21, 480)).astype(np.float32)
        return bida.LinearModelBackend("rc", W, 21, 0.5), lambda o, b: o.linear_evaluate(RC, W, 0.5, b)
    blob = make_bmlp1("rc", hidden=[128, 128], classes=21, ensemble=2, seed=12)
    return bida.MlpModelBackend("rc", blob, 0.5), lambda o, b: o.mlp_evaluate(blob, RC, 0.5, b, threads=8)


@pytest.mark.parametrize("model", ["linear", "mlp"])
def test_graph_replay_sizes_change(model):
    orc = Oracle()
    be, ref = backend(model)
    batches = [bida.random_walks("rc", n, 0, 30, seed=200 + i) for i, n in enumerate(SIZES)]
    want = [ref(orc, b) for b in batches]
    with be:
        g0 = be.graph_launch_count()
        for _ in range(3):  # every lane sees several sizes
            for b, w in zip(batches, want):
                assert (be.evaluate(b) == w).all()
            for t, w in zip([be.submit(b) for b in batches], want):
                assert (t.wait() == w).all()
        used = be.graph_launch_count() - g0
        assert used == 3 * 2 * len(SIZES), used


def test_graphs_off_matches(tmp_path):
    out = tmp_path / "h_off.npy"
    code = (
        "import numpy as np, paper_2507_11916_b200 as bida\n"
        "from paper_2507_11916_b200.models import make_bmlp1\n"
        "blob = make_bmlp1('rc', hidden=[128, 128], classes=21, ensemble=2, seed=12)\n"
        "b = bida.random_walks('rc', 5000, 0, 30, seed=3)\n"
        "with bida.MlpModelBackend('rc', blob, 0.5) as be:\n"
        "    h = be.evaluate(b); assert be.graph_launch_count() == 0\n"
        f"np.save({str(out)!r}, h)\n"
    )
    env = dict(os.environ, BIDA_GPU_GRAPHS="0")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    subprocess.run([sys.executable, "-c", code], env=env, cwd=root, check=True)
    h_off = np.load(out)
    blob = make_bmlp1("rc", hidden=[128, 128], classes=21, ensemble=2, seed=12)
    b = bida.random_walks("rc", 5000, 0, 30, seed=3)
    with bida.MlpModelBackend("rc", blob, 0.5) as be:
        assert (be.evaluate(b) == h_off).all()
        assert be.graph_launch_count() == 1
