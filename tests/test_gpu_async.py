"""Asynchronous submit / complete C-ABI (bida_gpu_submit, _batch_ready,
_batch_h, _batch_wait; SURVEY §8(b) optional extra): batches complete
independently and out of order, the GPU's h-values are readable in mapped host
memory once ready, and each batch reports only its own errors."""
import threading

import numpy as np
import pytest

import paper_2507_11916_b200 as bida
from oracle_lib import RC, Oracle
from paper_2507_11916_b200.models import make_bmlp1

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("model", ["linear", "mlp"])
def test_eight_in_flight_out_of_order(model):
    orc = Oracle()
    batches = [bida.random_walks("rc", n, 0, 30, seed=50 + i) for i, n in enumerate([1, 7, 128, 129, 1000, 4096, 32768, 300])]
    if model == "linear":
        W = np.random.default_rng(3).uniform(-0.1, 0.1, (2, 21, 480)).astype(np.float32)
        be = bida.LinearModelBackend("rc", W, 21, 0.5)
        want = [orc.linear_evaluate(RC, W, 0.5, b) for b in batches]
    else:
        blob = make_bmlp1("rc", hidden=[128, 128], classes=21, ensemble=1, seed=9)
        be = bida.MlpModelBackend("rc", blob, 0.5)
        want = [orc.mlp_evaluate(blob, RC, 0.5, b, threads=8) for b in batches]
    with be:
        toks = [be.submit(b) for b in batches]
        for t, w in zip(toks, want):
            while not t.ready():
                pass
            assert (t.peek() == w).all()  # straight from mapped host memory
        for t, w in reversed(list(zip(toks, want))):
            assert (t.wait() == w).all()
        assert (be.evaluate(batches[3]) == want[3]).all()  # lanes released


def test_async_errors_stay_with_their_batch():
    W = np.random.default_rng(4).uniform(-0.1, 0.1, (1, 21, 480)).astype(np.float32)
    good = bida.random_walks("rc", 500, 0, 30, seed=1)
    bad = good.copy()
    bad["hi"][3] = np.uint64(0xFFFFFFFFFFFF)
    want = Oracle().linear_evaluate(RC, W, 0.5, good)
    with bida.LinearModelBackend("rc", W, 21, 0.5) as be:
        tb, tg = be.submit(bad), be.submit(good)
        assert (tg.wait() == want).all()
        with pytest.raises(ValueError, match="outside"):
            tb.wait()
        with pytest.raises(ValueError):
            be.submit(np.zeros(40000, bida.instances.packed_dtype("rc")))  # > 32768: capacity


def test_async_from_many_threads():
    W = np.random.default_rng(5).uniform(-0.1, 0.1, (1, 21, 480)).astype(np.float32)
    batches = [bida.random_walks("rc", 256 + 17 * i, 0, 30, seed=90 + i) for i in range(16)]
    want = [Oracle().linear_evaluate(RC, W, 0.5, b) for b in batches]
    errors = []
    with bida.LinearModelBackend("rc", W, 21, 0.5) as be:
        # two threads x at most 4 batches in flight each: never more than the 8
        # lanes held at once (a caller holding lanes while waiting for more
        # could otherwise starve)
        def work(t):
            for r in range(20):
                idx = [i for i in range(t, 16, 2)][(r % 2) * 4:(r % 2) * 4 + 4]
                toks = [be.submit(batches[i]) for i in idx]
                for i, tk in zip(idx, toks):
                    if not (tk.wait() == want[i]).all():
                        errors.append(i)
        ths = [threading.Thread(target=work, args=(t,)) for t in range(2)]
        for th in ths:
            th.start()
        for th in ths:
            th.join()
    assert not errors


def test_begin_fill_launch_wait():
    """bida_gpu_batch_begin hands out the lane's mapped input buffer; the caller
    packs states straight into it (GpuBackend does), launch + wait complete it."""
    import ctypes as C

    from paper_2507_11916_b200 import _native

    W = np.random.default_rng(6).uniform(-0.1, 0.1, (1, 21, 480)).astype(np.float32)
    packed = bida.random_walks("rc", 777, 0, 30, seed=8)
    L = _native.lib()
    with bida.LinearModelBackend("rc", W, 21, 0.5) as be:
        b, buf = C.c_void_p(), C.c_void_p()
        _native.check(L.bida_gpu_batch_begin(be._h, len(packed), C.byref(b), C.byref(buf)))
        C.memmove(buf, packed.ctypes.data, packed.nbytes)
        _native.check(L.bida_gpu_batch_launch(b))
        h = np.empty(len(packed), np.int32)
        _native.check(L.bida_gpu_batch_wait(b, h.ctypes.data_as(C.c_void_p)))
    assert (h == Oracle().linear_evaluate(RC, W, 0.5, packed)).all()
