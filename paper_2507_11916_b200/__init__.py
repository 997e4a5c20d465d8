"""B200-native batched heuristic evaluator for Batch IDA* / CB-DFS
(arXiv 2507.11916): a drop-in for the reference's EvaluatorBackend.

Product code lives in csrc/ (CUDA + C-ABI, built into _lib/libbida_gpu.so);
this package is the Python host mirror of the reference's backend API.
"""
from .backend import (LinearModelBackend, MlpModelBackend, blin1_bytes, pdb_build, pdb_build_save,  # noqa: F401
                      random_walks_device, random_walks_fast)
from .instances import ACTIVE, FEATURES, PACKED_BYTES, RC, STP2, STP3, STP4, domain_id, random_walks  # noqa: F401

__all__ = [
    "LinearModelBackend",
    "MlpModelBackend",
    "blin1_bytes",
    "random_walks",
    "domain_id",
]
