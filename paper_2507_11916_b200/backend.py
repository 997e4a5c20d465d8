"""Python host mirror of the reference's evaluator backends, on the B200.

Mirrors bida::LinearModelBackend<D> (batch_eval.hpp:82-187) — constructor
checks, BLIN1 load/save, evaluate over a batch, needs_features — but the batch
is a numpy array of PACKED states (stp.hpp:121-126 / rubiks.hpp:126-137) and
evaluation runs in the CUDA library through the C-ABI (include/bida_gpu.h).
`MlpModelBackend` is the same interface for the project's BMLP1 integer MLP
(the reference has no MLP).

Errors raise ValueError where the reference throws std::invalid_argument and
RuntimeError where it throws std::runtime_error.
"""
from __future__ import annotations

import ctypes as C
import struct

import numpy as np

from . import _native
from .instances import FEATURES, domain_id, packed_dtype


def _as_packed(domain: int, packed) -> np.ndarray:
    """Accepts the packed dtype, u64[n] (STP) or u64[n][2] (Rubik's lo, hi)."""
    a = np.ascontiguousarray(packed)
    want = packed_dtype(domain)
    if a.dtype == want:
        return a
    if a.dtype == np.uint64 and a.ndim == 2 and a.shape[1] * 8 == want.itemsize:
        return a.view(want).reshape(-1)
    if a.dtype == np.uint64 and a.ndim == 1 and want.itemsize == 8:
        return a
    raise ValueError(f"packed states must be {want} (got {a.dtype} {a.shape})")


class _GpuBackendBase:
    _h = None

    def __init__(self) -> None:
        self._h = None

    # --- EvaluatorBackend<D> interface (batch_eval.hpp:45-51) ---------------
    def needs_features(self) -> bool:
        """The GPU encodes on the device from packed states."""
        return False

    def evaluate(self, packed, out: np.ndarray | None = None) -> np.ndarray:
        """h-values (int32) for a batch of packed states (batch_eval.hpp:49).
        `out` (optional, int32[n]) receives the result; page-locked host
        buffers on either side are transferred by DMA without staging."""
        p = _as_packed(self.domain, packed)
        if out is None:
            h = np.empty(len(p), np.int32)
        else:
            h = out
            if h.dtype != np.int32 or not h.flags["C_CONTIGUOUS"] or len(h) != len(p):
                raise ValueError("out must be a contiguous int32 array of the batch length")
        if len(p):
            _native.check(
                _native.lib().bida_gpu_evaluate(self._h, p.ctypes.data_as(C.c_void_p), len(p),
                                                h.ctypes.data_as(C.c_void_p))
            )
        return h

    def submit(self, packed) -> "Batch":
        """Asynchronous evaluation of <= 32768 states (bida_gpu_submit): returns
        a Batch whose ready() / wait() complete it; up to 8 in flight."""
        p = np.ascontiguousarray(_as_packed(self.domain, packed))
        b = C.c_void_p()
        _native.check(_native.lib().bida_gpu_submit(self._h, p.ctypes.data_as(C.c_void_p), len(p), C.byref(b)))
        return Batch(b, len(p))

    def evaluate_logits(self, packed):
        """(h, logits[n][E][C] float64): diagnostics for parity tests."""
        p = _as_packed(self.domain, packed)
        info = self.info()
        h = np.empty(len(p), np.int32)
        lg = np.empty((len(p), info.ensemble, info.classes), np.float64)
        if len(p):
            _native.check(
                _native.lib().bida_gpu_evaluate_logits(
                    self._h, p.ctypes.data_as(C.c_void_p), len(p), h.ctypes.data_as(C.c_void_p),
                    lg.ctypes.data_as(C.c_void_p))
            )
        return h, lg

    def evaluate_device(self, d_packed, d_h, n: int | None = None, d_logits=None, stream=None) -> None:
        """Asynchronous device-resident evaluation: torch CUDA tensors (or raw
        device pointers) in, h written into d_h on `stream` (default: torch's
        current stream).  Call `status()` after synchronising."""
        def ptr(t):
            if t is None:
                return None
            return C.c_void_p(t if isinstance(t, int) else t.data_ptr())
        if n is None:
            n = d_h.numel()
        if stream is None:
            import torch

            stream = torch.cuda.current_stream().cuda_stream
        elif not isinstance(stream, int):
            stream = stream.cuda_stream
        _native.check(
            _native.lib().bida_gpu_evaluate_device(self._h, ptr(d_packed), n, ptr(d_h), ptr(d_logits),
                                                   C.c_void_p(stream))
        )

    def attach_pdb(self, pattern, entries=None, mode: str = "min", path: str | None = None) -> None:
        """PDB correction in the readout: h = min(h_model, h_PDB) ("min") or
        h_PDB with the model still evaluated ("replace", PAPER.md:407 Table-1
        mode); "off" detaches.  `entries` as PdbTable::entries() (pdb.hpp), or a
        BPDB1 file via `path`."""
        m = {"off": _native.PDB_OFF, "min": _native.PDB_MIN, "replace": _native.PDB_REPLACE}[mode]
        L = _native.lib()
        if entries is None and path is None and m != _native.PDB_OFF:
            # build the table on this handle's device (bida_gpu_attach_pdb_built)
            pat = np.ascontiguousarray(pattern, np.uint8)
            _native.check(L.bida_gpu_attach_pdb_built(self._h, pat.ctypes.data_as(C.c_void_p), len(pat), m))
            return
        if path is not None:
            _native.check(L.bida_gpu_attach_pdb_file(self._h, str(path).encode(), m))
            return
        pat = np.ascontiguousarray(pattern if pattern is not None else [], np.uint8)
        ent = np.ascontiguousarray(entries if entries is not None else [], np.uint8)
        _native.check(L.bida_gpu_attach_pdb(self._h, pat.ctypes.data_as(C.c_void_p), len(pat),
                                            ent.ctypes.data_as(C.c_void_p), len(ent), m))

    def status(self) -> None:
        _native.check(_native.lib().bida_gpu_stream_status(self._h))

    def info(self) -> _native.ModelInfo:
        out = _native.ModelInfo()
        _native.check(_native.lib().bida_gpu_info(self._h, C.byref(out)))
        return out

    def exact_replays(self) -> int:
        """(state, member) readouts so far that took the exact float64 replay
        because the certified float32 bound could not decide (parity evidence)."""
        v = C.c_int64(0)
        _native.check(_native.lib().bida_gpu_exact_replays(self._h, C.byref(v)))
        return int(v.value)

    def launch_count(self) -> int:
        return int(_native.lib().bida_gpu_launch_count(self._h))

    def graph_launch_count(self) -> int:
        """Launches that replayed a zero-copy lane's CUDA graph."""
        return int(_native.lib().bida_gpu_graph_launch_count(self._h))

    def close(self) -> None:
        if self._h:
            _native.lib().bida_gpu_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


class LinearModelBackend(_GpuBackendBase):
    """GPU drop-in for bida::LinearModelBackend<D> (batch_eval.hpp:82-187).

    member_weights: E arrays of C*F floats (row-major [C][F]) or one array
    shaped [E][C][F]; classes: C; quantile: q of quantile_class.
    """

    def __init__(self, domain, member_weights, classes: int, quantile: float, device: int = 0):
        super().__init__()
        self.domain = domain_id(domain)
        F = FEATURES[self.domain]
        ws = [np.asarray(w, np.float32).reshape(-1) for w in member_weights]
        if not ws:
            raise ValueError("LinearModelBackend: empty ensemble")
        if classes <= 0:
            raise ValueError("LinearModelBackend: need at least one class")
        for w in ws:
            if w.size != classes * F:
                raise ValueError("LinearModelBackend: weight matrix size mismatch")
        W = np.ascontiguousarray(np.stack(ws))
        h = C.c_void_p()
        _native.check(
            _native.lib().bida_gpu_linear_create(device, self.domain, W.ctypes.data_as(C.c_void_p),
                                                 len(ws), classes, float(quantile), C.byref(h))
        )
        self._h = h
        self.classes, self.quantile, self.ensemble = classes, float(quantile), len(ws)

    @classmethod
    def load(cls, domain, path: str, quantile: float, device: int = 0) -> "LinearModelBackend":
        """LinearModelBackend::load (batch_eval.hpp:109-131)."""
        self = cls.__new__(cls)
        _GpuBackendBase.__init__(self)
        self.domain = domain_id(domain)
        h = C.c_void_p()
        _native.check(_native.lib().bida_gpu_linear_load(device, self.domain, str(path).encode(),
                                                         float(quantile), C.byref(h)))
        self._h = h
        info = self.info()
        self.classes, self.quantile, self.ensemble = info.classes, float(quantile), info.ensemble
        return self

    @staticmethod
    def save(domain, path: str, weights, classes: int) -> None:
        """LinearModelBackend::save (batch_eval.hpp:133-145): BLIN1 image."""
        d = domain_id(domain)
        with open(path, "wb") as f:
            f.write(blin1_bytes(d, weights, classes))


def blin1_bytes(domain, weights, classes: int) -> bytes:
    d = domain_id(domain)
    ws = [np.asarray(w, np.float32).reshape(-1) for w in weights]
    head = b"BLIN1" + struct.pack("<III", FEATURES[d], classes, len(ws))
    return head + b"".join(w.astype("<f4").tobytes() for w in ws)


class MlpModelBackend(_GpuBackendBase):
    """The BMLP1 integer MLP ensemble behind the same API."""

    def __init__(self, domain, blob: bytes, quantile: float, device: int = 0):
        super().__init__()
        self.domain = domain_id(domain)
        b = np.frombuffer(bytes(blob), np.uint8)
        h = C.c_void_p()
        _native.check(
            _native.lib().bida_gpu_mlp_create_bmlp1(device, self.domain, b.ctypes.data_as(C.c_void_p),
                                                    len(b), float(quantile), C.byref(h))
        )
        self._h = h
        info = self.info()
        self.classes, self.quantile, self.ensemble = info.classes, float(quantile), info.ensemble

    @classmethod
    def load(cls, domain, path: str, quantile: float, device: int = 0) -> "MlpModelBackend":
        with open(path, "rb") as f:
            return cls(domain, f.read(), quantile, device)


class Batch:
    """An in-flight asynchronous batch (bida_gpu_submit)."""

    def __init__(self, handle, n):
        self._b, self.n = handle, n

    def ready(self) -> bool:
        r = _native.lib().bida_gpu_batch_ready(self._b)
        if r < 0:
            _native.check(-r)
        return r == 1

    def peek(self) -> np.ndarray:
        """The h-values in mapped host memory where the GPU wrote them (valid
        once ready(), until wait())."""
        ptr = _native.lib().bida_gpu_batch_h(self._b)
        return np.ctypeslib.as_array(ptr, shape=(self.n,)).copy() if self.n else np.empty(0, np.int32)

    def wait(self) -> np.ndarray:
        if self._b is None:
            raise RuntimeError("batch already completed")
        h = np.empty(self.n, np.int32)
        b, self._b = self._b, None
        _native.check(_native.lib().bida_gpu_batch_wait(b, h.ctypes.data_as(C.c_void_p)))
        return h


def pdb_build(domain, pattern, device: int = 0, max_entries: int = 0) -> np.ndarray:
    """PdbTable<D>::build(pattern, D::solved()) (pdb.hpp:30-64) on the GPU:
    the entries (uint8; 0xFF unreachable), byte-identical to the reference's."""
    L = _native.lib()
    d = domain_id(domain)
    pat = np.ascontiguousarray(pattern, np.uint8)
    n = C.c_uint64(0)
    rc = L.bida_gpu_pdb_build(device, d, pat.ctypes.data_as(C.c_void_p), len(pat), max_entries, None, 0,
                              C.byref(n), None)
    if rc != _native.BIDA_ERR_CAPACITY:
        _native.check(rc)
    out = np.empty(n.value, np.uint8)
    depth = C.c_int(0)
    _native.check(L.bida_gpu_pdb_build(device, d, pat.ctypes.data_as(C.c_void_p), len(pat), max_entries,
                                       out.ctypes.data_as(C.c_void_p), n.value, C.byref(n), C.byref(depth)))
    return out


def pdb_build_save(domain, pattern, path: str, device: int = 0) -> None:
    """Same, written as a BPDB1 file (PdbTable::save, pdb.hpp:78-96)."""
    pat = np.ascontiguousarray(pattern, np.uint8)
    _native.check(_native.lib().bida_gpu_pdb_build_save(device, domain_id(domain), pat.ctypes.data_as(C.c_void_p),
                                                        len(pat), str(path).encode()))


def random_walks_device(domain, n: int, len_min: int = 0, len_max: int = 30, seed: int = 0, device: int = 0):
    """n packed random-walk scrambles generated on the GPU (bida_gpu_random_walks)
    as a torch uint8 CUDA tensor of n * packed-bytes (synthetic benchmark input;
    `random_walks` is the numpy equivalent with a different RNG)."""
    import torch

    d = domain_id(domain)
    pb = 16 if d == 100 else 8
    out = torch.empty(n * pb, dtype=torch.uint8, device=torch.device("cuda", device))
    stream = torch.cuda.current_stream(device).cuda_stream
    _native.check(_native.lib().bida_gpu_random_walks(device, d, n, len_min, len_max, seed,
                                                      C.c_void_p(out.data_ptr()), C.c_void_p(stream)))
    return out


def random_walks_fast(domain, n: int, len_min: int = 0, len_max: int = 30, seed: int = 0, device: int = 0):
    """Same, copied to a host numpy array of packed states."""
    t = random_walks_device(domain, n, len_min, len_max, seed, device)
    return t.cpu().numpy().view(packed_dtype(domain))
