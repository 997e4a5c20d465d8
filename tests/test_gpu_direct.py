"""C-ABI direct path (bida_gpu.cu, bida_gpu_evaluate): page-locked caller
buffers are mapped into the device's address space, so one kernel launch reads
the packed states over PCIe and writes h straight back.  Results must equal
the chunked copy pipeline (pageable buffers) and the oracle; misaligned or
pageable buffers must take the pipeline; errors still reach the caller."""
import numpy as np
import pytest
import torch

import paper_2507_11916_b200 as bida
from oracle_lib import DOMAINS, Oracle
from paper_2507_11916_b200.models import make_bmlp1

pytestmark = pytest.mark.gpu
FEAT = {"rc": 480, "stp4": 256, "stp3": 81}


def pinned(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.uint8).copy()).pin_memory().numpy().view(a.dtype)


def pinned_out(n):
    return torch.empty(n, dtype=torch.int32).pin_memory().numpy()


def make(domain, kind):
    if kind == "linear":
        W = np.random.default_rng(7).uniform(-0.1, 0.1, (2, 24, FEAT[domain])).astype(np.float32)
        return bida.LinearModelBackend(domain, W, 24, 0.5), lambda o, p: o.linear_evaluate(DOMAINS[domain], W, 0.5, p)
    blob = make_bmlp1(domain, hidden=[128, 128], classes=24, ensemble=1, seed=8)
    return bida.MlpModelBackend(domain, blob, 0.5), lambda o, p: o.mlp_evaluate(blob, DOMAINS[domain], 0.5, p, threads=8)


@pytest.mark.parametrize("domain", ["rc", "stp4", "stp3"])
@pytest.mark.parametrize("kind", ["linear", "mlp"])
def test_direct_matches_pipeline_and_oracle(domain, kind):
    n = 600_011  # > 2^18: the copy pipeline takes several chunks, the direct path one launch
    packed = bida.random_walks(domain, n, 0, 60, seed=31)
    be, ref = make(domain, kind)
    with be:
        h_pipe = be.evaluate(packed)  # pageable: copy pipeline
        hp, ho = pinned(packed), pinned_out(n)
        l0 = be.launch_count()
        be.evaluate(hp, out=ho)
        assert be.launch_count() - l0 == 1  # one launch over mapped host memory
        assert (ho == h_pipe).all()
        sample = np.ascontiguousarray(packed[::97])
        assert (h_pipe[::97] == ref(Oracle(), sample)).all()


def test_misaligned_pinned_buffer_takes_the_pipeline():
    n = 100_000
    packed = bida.random_walks("rc", n, 0, 30, seed=4)
    be, _ = make("rc", "mlp")
    raw = torch.empty((n + 1) * 16, dtype=torch.uint8).pin_memory().numpy()
    view = raw[8:8 + n * 16]  # 8-byte aligned: not a valid 16-byte state load
    view[:] = packed.view(np.uint8)
    with be:
        want = be.evaluate(packed)
        got = be.evaluate(view.view(packed.dtype))
        assert (got == want).all()


def test_direct_path_reports_bad_states():
    n = 70_000
    packed = bida.random_walks("rc", n, 0, 30, seed=5)
    packed["hi"][12345] = np.uint64(0xFFFFFFFFFFFF)
    be, _ = make("rc", "linear")
    hp, ho = pinned(packed), pinned_out(n)
    with be:
        with pytest.raises(ValueError, match="outside"):
            be.evaluate(hp, out=ho)
        good = bida.random_walks("rc", n, 0, 30, seed=6)
        assert (be.evaluate(pinned(good), out=pinned_out(n)) == be.evaluate(good)).all()  # error cleared
