"""Batch IDA* nodes/s with the B200 evaluator vs the reference CPU evaluator
(BASELINE.json metric, second half).  Runs tests/cpp/bin/search_parity (the
reference's own batch_idastar / aidastar with GpuBackend or
LinearModelBackend dropped in) on Korf's 15-puzzle instances with the
linear-Manhattan model and prints one JSON line
per run.  Not a pytest test; results are committed under profiles/.

    python tests/search_bench.py --instances 8,4 --threads 16
"""
import argparse
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
BIN = os.path.join(ROOT, "tests", "cpp", "bin", "search_parity")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--instances", default="8,4")  # korf10 indices (0-based): #9 cost 46, #5 cost 56
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 8)
    ap.add_argument("--out", default="")
    ap.add_argument("--domain", default="stp4", choices=["stp4", "rc"])
    ap.add_argument("--time-limit", type=float, default=30.0)
    ap.add_argument("--walks", default="3:14:16:2507")  # rc: n:len_min:len_max:seed
    a = ap.parse_args()
    if a.domain == "rc":
        return rc_bench(a)
    from oracle_lib import manhattan_linear_weights

    import paper_2507_11916_b200 as bida

    g = np.load(os.path.join(ROOT, "tests", "golden", "instances.npz"))
    inst = "/tmp/korf10.txt"
    with open(inst, "w") as f:
        for v in g["korf10"]:
            v = int(v)
            f.write("stp 4 " + " ".join(str((v >> (4 * c)) & 15) for c in range(16)) + "\n")
    blin = "/tmp/man4.blin"
    open(blin, "wb").write(bida.blin1_bytes("stp4", manhattan_linear_weights(4, 72, 4.0), 72))
    n = a.threads
    runs = [
        # (label, mode, extra args)
        ("gpu batch_idastar E=1", "gpu", ["--evaluators", "1", "--work-num", "32", "--batch", "8192", "--timeout-us", "100"]),
        ("gpu batch_idastar E=4", "gpu", ["--evaluators", "4", "--work-num", "32", "--batch", "4096", "--timeout-us", "100"]),
        ("cpu batch_idastar E=n", "cpu", ["--evaluators", str(n), "--work-num", "8", "--batch", "256", "--timeout-us", "100"]),
        ("cpu aidastar (immediate)", "cpu", ["--immediate", "--evaluators", "1", "--work-num", "1", "--batch", "1"]),
    ]
    lines = []
    for idx in a.instances.split(","):
        for label, mode, extra in runs:
            cmd = [BIN, "--domain", "stp4", "--instances", inst, "--model", "linear:" + blin, "--mode", mode,
                   "--threads", str(n), "--first", idx, "--count", "1", *extra]
            out = subprocess.run(cmd, capture_output=True, text=True, timeout=1800)
            if out.returncode:
                print(out.stderr, file=sys.stderr)
                continue
            for l in out.stdout.splitlines():
                if l.startswith("{"):
                    r = json.loads(l)
                    r["label"] = label
                    r.pop("iterations", None)
                    lines.append(r)
                    print(json.dumps(r), flush=True)
    if a.out:
        with open(a.out, "w") as f:
            for r in lines:
                f.write(json.dumps(r) + "\n")


def rc_bench(a):
    """Config 2 (BASELINE.json): Rubik's Batch IDA*, walks 14-16, BMLP1 480-128-128-21
    evaluated per node on the GPU (or by the oracle on the CPU), search guided
    by the reference's 5-corner PDB (Table-1 mode).  Each run is
    time-limited; nodes/s is generated / wall."""
    from paper_2507_11916_b200.models import make_bmlp1

    model = "/tmp/m128.bmlp"
    open(model, "wb").write(make_bmlp1("rc", hidden=[128, 128], classes=21, seed=2507))
    n = a.threads
    tl = str(a.time_limit)
    runs = [
        ("gpu batch_idastar nn+gpu-pdb E=1", "gpu", ["--gpu-pdb", "--evaluators", "1", "--work-num", "64", "--batch", "16384", "--timeout-us", "200"]),
        ("gpu batch_idastar nn+gpu-pdb E=2", "gpu", ["--gpu-pdb", "--evaluators", "2", "--work-num", "64", "--batch", "8192", "--timeout-us", "200"]),
        ("gpu batch_idastar nn+gpu-pdb E=4", "gpu", ["--gpu-pdb", "--evaluators", "4", "--work-num", "64", "--batch", "8192", "--timeout-us", "200"]),
        ("gpu batch_idastar nn+cpu-pdb E=2", "gpu", ["--evaluators", "2", "--work-num", "64", "--batch", "8192", "--timeout-us", "200"]),
        ("cpu batch_idastar nn+pdb E=n", "cpu", ["--evaluators", str(n), "--work-num", "8", "--batch", "512", "--timeout-us", "200"]),
        ("cpu aidastar nn+pdb (immediate)", "cpu", ["--immediate", "--evaluators", "1", "--work-num", "1", "--batch", "1"]),
        ("cpu aidastar pdb only (no nn)", "pdb", ["--immediate", "--evaluators", "1", "--work-num", "1", "--batch", "1"]),
    ]
    lines = []
    only = os.environ.get("BIDA_SEARCH_ONLY")  # e.g. "gpu" to rerun just the GPU rows
    for label, mode, extra in runs:
        if only and not label.startswith(only):
            continue
        cmd = [BIN, "--domain", "rc", "--walks", a.walks, "--model", "mlp:" + model, "--mode", mode,
               "--table1-pdb", "5", "--threads", str(n), "--time-limit", tl, *extra]
        out = subprocess.run(cmd, capture_output=True, text=True, timeout=3600)
        if out.returncode:
            print(out.stderr, file=sys.stderr)
            continue
        for l in out.stdout.splitlines():
            if l.startswith("{"):
                r = json.loads(l)
                r["label"] = label
                r.pop("iterations", None)
                lines.append(r)
                print(json.dumps(r), flush=True)
    if a.out:
        with open(a.out, "w") as f:
            for r in lines:
                f.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
