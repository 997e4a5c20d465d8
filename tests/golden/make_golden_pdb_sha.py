"""Digests of pattern databases built BY THE REFERENCE (PdbTable<D>::build +
save, pdb.hpp:30-96, through oracle/_ref) that are too large to commit: the
sha256 of the BPDB1 file and the per-depth entry histogram.  The GPU builder
(bida_gpu_pdb_build_save) must reproduce the file byte for byte
(tests/test_gpu_pdb_build.py).  The 7- and 8-corner Rubik's tables take ~10
minutes each on one core here.

    python tests/golden/make_golden_pdb_sha.py [corners ...]
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle_lib import RC, RefLib  # noqa: E402

OUT = os.path.join(HERE, "pdb_rc_digests.json")


def main(corners):
    ref = RefLib()
    digests = json.load(open(OUT)) if os.path.exists(OUT) else {}
    for m in corners:
        path = f"/tmp/bida_ref_rc_c{m}.pdb"
        t0 = time.time()
        ref.pdb_build_save(RC, list(range(m)), path)
        data = open(path, "rb").read()
        ent = np.frombuffer(data, np.uint8, offset=8 + m + 8)
        hist = np.bincount(ent, minlength=256)
        digests[f"rc_c{m}"] = {
            "pattern": list(range(m)), "file_bytes": len(data), "entries": int(len(ent)),
            "sha256": hashlib.sha256(data).hexdigest(),
            "depth_histogram": {str(d): int(c) for d, c in enumerate(hist) if c},
            "reference_build_seconds": round(time.time() - t0, 1),
        }
        print(m, digests[f"rc_c{m}"]["sha256"], flush=True)
        json.dump(digests, open(OUT, "w"), indent=1)


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [5, 6])
