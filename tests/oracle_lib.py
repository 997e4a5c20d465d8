"""ctypes bindings to the TEST-ONLY checkers under oracle/.

* ``Oracle``  -> oracle/_build/libbida_oracle.so, the plain-C restatement.
* ``RefLib``  -> oracle/_ref/libbida_ref.so, the reference's own headers
  compiled unchanged (built here from /root/reference; the prebuilt .so
  travels to the GPU box).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg use this.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
ORACLE_SO = os.path.join(ORACLE_DIR, "_build", "libbida_oracle.so")
REF_SO = os.path.join(ORACLE_DIR, "_ref", "libbida_ref.so")

STP2, STP3, STP4, RC = 2, 3, 4, 100
DOMAINS = {"stp2": STP2, "stp3": STP3, "stp4": STP4, "rc": RC}
FEATURES = {STP2: 16, STP3: 81, STP4: 256, RC: 480}
PACKED_BYTES = {STP2: 8, STP3: 8, STP4: 8, RC: 16}

_p = C.c_void_p
_i64 = C.c_int64


def _ptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(C.c_void_p)


def packed_dtype(domain: int):
    """Packed states are u64 (STP) or two u64 {lo, hi} (RC) per state."""
    return np.dtype("<u8") if domain != RC else np.dtype([("lo", "<u8"), ("hi", "<u8")])


def ensure_built() -> None:
    """Build the checkers if missing (needs /root/reference for _ref)."""
    if not os.path.exists(ORACLE_SO) or (
        not os.path.exists(REF_SO) and os.path.isdir("/root/reference/proj/include")
    ):
        subprocess.run(["make", "-s", "-C", ORACLE_DIR], check=True)


class Oracle:
    def __init__(self) -> None:
        ensure_built()
        L = C.CDLL(ORACLE_SO)
        L.orc_encode.argtypes = [C.c_int, _p, _i64, _p]
        L.orc_linear_evaluate.argtypes = [C.c_int, _p, C.c_int, C.c_int, C.c_double, _p, _i64, _p, _p]
        L.orc_quantile_class.argtypes = [_p, C.c_int, C.c_double, C.POINTER(C.c_int)]
        L.orc_active_indices.argtypes = [C.c_int, _p, _p]
        L.orc_mlp_evaluate_blob.argtypes = [_p, C.c_size_t, C.c_int, C.c_double, _p, _i64, _p, _p, C.c_int]
        L.orc_manhattan.argtypes = [C.c_int, _p, _i64, _p]
        L.orc_pdb_lookup.argtypes = [C.c_int, _p, C.c_int, _p, C.c_uint64, _p, _i64, _p]
        L.orc_blin1_parse.argtypes = [_p, C.c_size_t, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.POINTER(C.c_float))]
        self.L = L

    def encode(self, domain, packed):
        out = np.zeros((len(packed), FEATURES[domain]), np.float32)
        assert self.L.orc_encode(domain, _ptr(packed), len(packed), _ptr(out)) == 0
        return out

    def active_indices(self, domain, packed_one):
        idx = np.zeros(32, np.int32)
        k = self.L.orc_active_indices(domain, _ptr(packed_one), _ptr(idx))
        return idx[:k]

    def linear_evaluate(self, domain, W, q, packed, want_logits=False):
        W = np.ascontiguousarray(W, np.float32)
        E, Cc, F = W.shape
        h = np.zeros(len(packed), np.int32)
        lg = np.zeros((len(packed), E, Cc), np.float64) if want_logits else None
        rc = self.L.orc_linear_evaluate(domain, _ptr(W), E, Cc, q, _ptr(packed), len(packed), _ptr(h), _ptr(lg))
        if rc != 0:
            raise ValueError(f"oracle error {rc}")
        return (h, lg) if want_logits else h

    def mlp_evaluate(self, blob: bytes, domain, q, packed, want_logits=False, E=None, Cc=None, threads=1):
        b = np.frombuffer(blob, np.uint8).copy()
        h = np.zeros(len(packed), np.int32)
        lg = np.zeros((len(packed), E, Cc), np.float64) if want_logits else None
        rc = self.L.orc_mlp_evaluate_blob(_ptr(b), len(b), domain, q, _ptr(packed), len(packed), _ptr(h), _ptr(lg), threads)
        if rc != 0:
            raise ValueError(f"oracle error {rc}")
        return (h, lg) if want_logits else h

    def quantile_class(self, p, q):
        p = np.ascontiguousarray(p, np.float64)
        err = C.c_int(0)
        c = self.L.orc_quantile_class(_ptr(p), len(p), q, C.byref(err))
        if err.value:
            raise ValueError("invalid quantile/distribution")
        return c

    def manhattan(self, domain, packed):
        out = np.zeros(len(packed), np.int32)
        assert self.L.orc_manhattan(domain, _ptr(packed), len(packed), _ptr(out)) == 0
        return out

    def pdb_lookup(self, domain, pattern, entries, packed):
        pat = np.ascontiguousarray(pattern, np.uint8)
        ent = np.ascontiguousarray(entries, np.uint8)
        out = np.zeros(len(packed), np.int32)
        rc = self.L.orc_pdb_lookup(domain, _ptr(pat), len(pat), _ptr(ent), len(ent), _ptr(packed), len(packed), _ptr(out))
        if rc:
            raise ValueError("invalid state for the pattern")
        return out


class RefLib:
    """The reference implementation itself (header-only C++ compiled unchanged)."""

    def __init__(self) -> None:
        ensure_built()
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(REF_SO)
        L = C.CDLL(REF_SO)
        L.ref_last_error.restype = C.c_char_p
        L.ref_random_walk_packed.argtypes = [C.c_int, _i64, C.c_int, C.c_int, C.c_uint64, _p]
        L.ref_repack.argtypes = [C.c_int, _p, _i64, _p]
        L.ref_encode.argtypes = [C.c_int, _p, _i64, _p]
        L.ref_linear_evaluate.argtypes = [C.c_int, _p, C.c_int, C.c_int, C.c_double, _p, _i64, _p, C.c_int]
        L.ref_linear_prepare.argtypes = [C.c_int, _p, C.c_int, C.c_int, C.c_double, _p, _i64]
        L.ref_linear_prepare.restype = C.c_void_p
        L.ref_linear_run.argtypes = [C.c_void_p, _p, C.c_int]
        L.ref_linear_release.argtypes = [C.c_void_p]
        L.ref_blin1_save.argtypes = [C.c_int, C.c_char_p, _p, C.c_int, C.c_int]
        L.ref_blin1_load_evaluate.argtypes = [C.c_int, C.c_char_p, C.c_double, _p, _i64, _p]
        L.ref_quantile_class.argtypes = [_p, C.c_int, C.c_double, C.POINTER(C.c_int)]
        L.ref_ensemble_min.argtypes = [_p, C.c_int, C.POINTER(C.c_int)]
        L.ref_manhattan.argtypes = [C.c_int, _p, _i64, _p]
        L.ref_pdb_build.argtypes = [C.c_int, _p, C.c_int, _p, C.c_uint64, C.POINTER(C.c_uint64)]
        L.ref_pdb_lookup_file.argtypes = [C.c_int, C.c_char_p, _p, _i64, _p]
        L.ref_pdb_build_save.argtypes = [C.c_int, _p, C.c_int, C.c_char_p]
        L.ref_load_instances.argtypes = [C.c_int, C.c_char_p, _p, _i64, C.POINTER(_i64)]
        L.ref_readout_scaled_logits.argtypes = [C.c_int, _p, _p, C.c_int, C.c_int, C.c_double, _i64, _p, C.c_int]
        self.L = L

    def _check(self, rc):
        if rc != 0:
            msg = self.L.ref_last_error().decode()
            raise (ValueError if rc in (1, 2) else RuntimeError)(msg)

    def random_walks(self, domain, n, len_min, len_max, seed):
        out = np.zeros(n, packed_dtype(domain))
        self._check(self.L.ref_random_walk_packed(domain, n, len_min, len_max, seed, _ptr(out)))
        return out

    def repack(self, domain, packed):
        out = np.zeros_like(packed)
        self._check(self.L.ref_repack(domain, _ptr(packed), len(packed), _ptr(out)))
        return out

    def encode(self, domain, packed):
        out = np.zeros((len(packed), FEATURES[domain]), np.float32)
        self._check(self.L.ref_encode(domain, _ptr(packed), len(packed), _ptr(out)))
        return out

    def linear_evaluate(self, domain, W, q, packed, threads=1):
        W = np.ascontiguousarray(W, np.float32)
        E, Cc, F = W.shape
        h = np.zeros(len(packed), np.int32)
        self._check(self.L.ref_linear_evaluate(domain, _ptr(W), E, Cc, q, _ptr(packed), len(packed), _ptr(h), threads))
        return h

    def blin1_save(self, domain, path, W):
        W = np.ascontiguousarray(W, np.float32)
        E, Cc, F = W.shape
        self._check(self.L.ref_blin1_save(domain, path.encode(), _ptr(W), E, Cc))

    def blin1_load_evaluate(self, domain, path, q, packed):
        h = np.zeros(len(packed), np.int32)
        self._check(self.L.ref_blin1_load_evaluate(domain, path.encode(), q, _ptr(packed), len(packed), _ptr(h)))
        return h

    def quantile_class(self, p, q):
        p = np.ascontiguousarray(p, np.float64)
        out = C.c_int(-1)
        self._check(self.L.ref_quantile_class(_ptr(p), len(p), q, C.byref(out)))
        return out.value

    def ensemble_min(self, v):
        v = np.ascontiguousarray(v, np.int32)
        out = C.c_int(-1)
        self._check(self.L.ref_ensemble_min(_ptr(v), len(v), C.byref(out)))
        return out.value

    def manhattan(self, domain, packed):
        out = np.zeros(len(packed), np.int32)
        self._check(self.L.ref_manhattan(domain, _ptr(packed), len(packed), _ptr(out)))
        return out

    def pdb_build(self, domain, pattern, cap=1 << 26):
        """PdbTable<D>::build (pdb.hpp:30-64) -> entries (uint8)."""
        pat = np.ascontiguousarray(pattern, np.uint8)
        buf = np.zeros(cap, np.uint8)
        n = C.c_uint64(0)
        self._check(self.L.ref_pdb_build(domain, _ptr(pat), len(pat), _ptr(buf), cap, C.byref(n)))
        return buf[: n.value].copy()

    def pdb_build_save(self, domain, pattern, path):
        pat = np.ascontiguousarray(pattern, np.uint8)
        self._check(self.L.ref_pdb_build_save(domain, _ptr(pat), len(pat), path.encode()))

    def pdb_lookup_file(self, domain, path, packed):
        """PdbTable<D>::load + lookup (pdb.hpp:66-69, 98-138)."""
        out = np.zeros(len(packed), np.int32)
        self._check(self.L.ref_pdb_lookup_file(domain, path.encode(), _ptr(packed), len(packed), _ptr(out)))
        return out

    def readout_scaled_logits(self, domain, acc, scale, q, threads=1):
        """The reference's LinearModelBackend::evaluate readout (softmax,
        quantile_class, ensemble_min) on logits (double)acc * (double)scale;
        acc int32 [n][E][C], scale float32 [E] (ref_harness.cpp)."""
        acc = np.ascontiguousarray(acc, np.int32)
        scale = np.ascontiguousarray(scale, np.float32)
        n, E, Cc = acc.shape
        h = np.zeros(n, np.int32)
        self._check(self.L.ref_readout_scaled_logits(domain, _ptr(acc), _ptr(scale), E, Cc, q, n, _ptr(h), threads))
        return h

    def load_instances(self, domain, path, cap=100000):
        out = np.zeros(cap, packed_dtype(domain))
        cnt = _i64(0)
        self._check(self.L.ref_load_instances(domain, path.encode(), _ptr(out), cap, C.byref(cnt)))
        return out[: min(cap, cnt.value)].copy()


def manhattan_linear_weights(N: int, classes: int = 72, alpha: float = 4.0) -> np.ndarray:
    """Linear-Manhattan weights: W[c][cell*K+t] =
    alpha*c*md(cell,t) - alpha*c^2/(2K); the softmax peaks at c = Manhattan."""
    K = N * N
    W = np.zeros((1, classes, K * K), np.float32)
    for c in range(classes):
        for cell in range(K):
            for t in range(K):
                md = 0 if t == 0 else abs(cell // N - t // N) + abs(cell % N - t % N)
                W[0, c, cell * K + t] = alpha * c * md - alpha * c * c / (2 * K)
    return W
