"""BMLP1: the integer-quantised MLP classifier ensemble.

The reference has no MLP; BMLP1 extends its BLIN1 linear
ensemble (batch_eval.hpp:107-131) to hidden layers while keeping the same
readout (softmax -> quantile_class -> ensemble_min).  Weights and activations
are integers (u8 activations, s8 weights) so that tensor-core 8-bit MMA with int32 accumulation computes the
logits exactly in any summation order — h is bit-exact by construction.

File layout (little-endian):
    "BMLP1", u32 F, u32 C, u32 E, u32 L, u32 H[L]
    per member, per layer l = 0..L (in = l ? H[l-1] : F, out = l < L ? H[l] : C):
        i8  W[out][in]  row-major
        i32 bias[out]
        u32 shift       (hidden layers only)
    per member: f32 out_scale
    hidden: a' = clamp((bias + W a) >> shift, 0, 255); output: logit = (bias + W a) * out_scale
"""
from __future__ import annotations

import struct
from dataclasses import dataclass, field

import numpy as np

from .instances import FEATURES, domain_id, random_walks


@dataclass
class Layer:
    W: np.ndarray          # int8 [out][in]
    bias: np.ndarray       # int32 [out]
    shift: int = 0         # hidden layers only


@dataclass
class BMLP1:
    F: int
    C: int
    hidden: list
    members: list = field(default_factory=list)   # list of (layers, out_scale)

    def to_bytes(self) -> bytes:
        out = [b"BMLP1", struct.pack("<IIII", self.F, self.C, len(self.members), len(self.hidden))]
        out += [struct.pack("<I", h) for h in self.hidden]
        for layers, scale in self.members:
            for li, ly in enumerate(layers):
                out.append(np.ascontiguousarray(ly.W, np.int8).tobytes())
                out.append(np.ascontiguousarray(ly.bias, "<i4").tobytes())
                if li < len(self.hidden):
                    out.append(struct.pack("<I", ly.shift))
            out.append(struct.pack("<f", scale))
        return b"".join(out)

    @staticmethod
    def from_bytes(blob: bytes) -> "BMLP1":
        if blob[:5] != b"BMLP1":
            raise RuntimeError("not a BMLP1 file")
        F, C, E, L = struct.unpack_from("<IIII", blob, 5)
        off = 21
        hidden = list(struct.unpack_from(f"<{L}I", blob, off))
        off += 4 * L
        m = BMLP1(F, C, hidden)
        dims = [F, *hidden, C]
        for _ in range(E):
            layers = []
            for li in range(L + 1):
                n_in, n_out = dims[li], dims[li + 1]
                W = np.frombuffer(blob, np.int8, n_in * n_out, off).reshape(n_out, n_in)
                off += n_in * n_out
                b = np.frombuffer(blob, "<i4", n_out, off)
                off += 4 * n_out
                s = 0
                if li < L:
                    (s,) = struct.unpack_from("<I", blob, off)
                    off += 4
                layers.append(Layer(W, b, s))
            (scale,) = struct.unpack_from("<f", blob, off)
            off += 4
            m.members.append((layers, scale))
        return m


def forward_int(layers, x: np.ndarray) -> np.ndarray:
    """Integer forward pass (int64 numpy) -> output accumulators [n][C]."""
    a = x.astype(np.int64)
    for li, ly in enumerate(layers):
        acc = a @ ly.W.astype(np.int64).T + ly.bias.astype(np.int64)
        if li < len(layers) - 1:
            a = np.clip(acc >> ly.shift, 0, 255)
        else:
            return acc
    return a


def _one_hot(domain: int, packed: np.ndarray) -> np.ndarray:
    F = FEATURES[domain]
    x = np.zeros((len(packed), F), np.int64)
    if domain == 100:
        lo, hi = packed["lo"].astype(np.uint64), packed["hi"].astype(np.uint64)
        rows = np.arange(len(packed))
        for p in range(8):
            c = (lo >> np.uint64(3 * p)) & np.uint64(7)
            co = (lo >> np.uint64(24 + 2 * p)) & np.uint64(3)
            x[rows, (c * np.uint64(24) + np.uint64(p * 3) + co).astype(np.int64)] = 1
        for p in range(12):
            e = (hi >> np.uint64(4 * p)) & np.uint64(15)
            eo = (lo >> np.uint64(40 + p)) & np.uint64(1)
            x[rows, (np.uint64(192) + e * np.uint64(24) + np.uint64(p * 2) + eo).astype(np.int64)] = 1
    else:
        N = domain
        K = N * N
        v = packed.astype(np.uint64)
        rows = np.arange(len(packed))
        for cell in range(K):
            t = ((v >> np.uint64(4 * cell)) & np.uint64(15)).astype(np.int64)
            x[rows, cell * K + t] = 1
    return x


def make_bmlp1(domain, hidden=(512, 512), classes: int = 21, ensemble: int = 1, seed: int = 0,
               logit_std: float = 2.5) -> bytes:
    """Seeded random BMLP1 model with calibrated shifts (activations use the
    0..255 range) and an output scale giving logits of std ~logit_std."""
    d = domain_id(domain)
    F = FEATURES[d]
    rng = np.random.default_rng(seed)
    sample = _one_hot(d, random_walks(d, 2048, 0, 30, seed=seed + 17))
    model = BMLP1(F, classes, list(hidden))
    dims = [F, *hidden, classes]
    for _ in range(ensemble):
        layers = []
        a = sample
        for li in range(len(dims) - 1):
            W = rng.integers(-127, 128, (dims[li + 1], dims[li]), dtype=np.int64).astype(np.int8)
            b = rng.integers(-512, 513, dims[li + 1]).astype(np.int32)
            acc = a @ W.astype(np.int64).T + b
            if li < len(dims) - 2:
                p = np.percentile(np.abs(acc), 95)
                shift = int(max(0, np.ceil(np.log2(max(p, 1) / 200.0))))
                layers.append(Layer(W, b, shift))
                a = np.clip(acc >> shift, 0, 255)
            else:
                layers.append(Layer(W, b, 0))
                sd = float(acc.std()) or 1.0
                scale = float(np.float32(logit_std / sd))
        model.members.append((layers, scale))
    return model.to_bytes()
