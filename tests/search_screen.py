"""Screens BASELINE config-2 instances (Rubik's random walks of 14-16 moves,
random_walk_instance, instance.hpp:36-57) for solved Table-1 search parity:
GPU Batch IDA* (network evaluated per node, h = 8-corner PDB on the device)
against the reference's CPU search with the same PDB (--mode pdb).  Writes one
JSON line per (length, seed, side) to gpurun_out/search_screen.jsonl.

    python tests/search_screen.py [--lengths 14,15,16] [--seeds 8] [--gpu-limit 60] [--cpu-limit 120]
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(exe, args, env=None, timeout=900):
    out = subprocess.run([os.path.join(ROOT, "tools", "bin", exe), *args], capture_output=True, text=True,
                         timeout=timeout, env={**os.environ, **(env or {})})
    rows = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    if out.returncode or not rows:
        return {"error": (out.stderr or "no output")[-300:]}
    return rows[0]


def main():
    from paper_2507_11916_b200.models import make_bmlp1

    ap = argparse.ArgumentParser()
    ap.add_argument("--lengths", default="14,15,16")
    ap.add_argument("--seeds", type=int, default=8)
    ap.add_argument("--seed0", type=int, default=2508)
    ap.add_argument("--gpu-limit", type=float, default=60)
    ap.add_argument("--cpu-limit", type=float, default=120)
    ap.add_argument("--corners", type=int, default=8)
    ap.add_argument("--exe", default="bida_search_fast")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "search_screen.jsonl"))
    ap.add_argument("--korf", default="", help="config 1 instead: comma-separated 0-based korf10 indices")
    args = ap.parse_args()
    if args.korf:
        return korf(args)
    model = "/tmp/bida_screen_h128.bmlp"
    with open(model, "wb") as f:
        f.write(make_bmlp1("rc", hidden=[128, 128], classes=21, ensemble=1, seed=2507))
    threads = str(len(os.sched_getaffinity(0)))
    common = ["--domain", "rc", "--model", "mlp:" + model, "--q", "0.5", "--table1-pdb", str(args.corners),
              "--pdb-build", "gpu", "--threads", threads, "--work-num", "128", "--batch", "16384",
              "--timeout-us", "25"]
    ring_env = {"BIDA_EVAL_AGENTS": "4", "BIDA_EVAL_SHARDS": "16"}
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    for L in [int(x) for x in args.lengths.split(",")]:
        for k in range(args.seeds):
            seed = args.seed0 + k
            walks = f"1:{L}:{L}:{seed}"
            g = run(args.exe, [*common, "--walks", walks, "--mode", "gpu", "--gpu-pdb", "--time-limit",
                               str(args.gpu_limit)], ring_env)
            row = {"length": L, "seed": seed, "side": "gpu", **g}
            with open(args.out, "a") as f:
                f.write(json.dumps(row) + "\n")
            print(L, seed, "gpu", g.get("status"), g.get("cost"), g.get("generated"), g.get("wall_s"), flush=True)
            if g.get("status") != "solved":
                continue
            c = run("bida_search", [*common, "--walks", walks, "--mode", "pdb", "--immediate",
                                    "--time-limit", str(args.cpu_limit)])
            row = {"length": L, "seed": seed, "side": "cpu_pdb", **c}
            same = (c.get("status") == "solved" and c["cost"] == g["cost"] and c["thresholds"] == g["thresholds"]
                    and [i[:3] for i in c["iterations"][:-1]] == [i[:3] for i in g["iterations"][:-1]])
            row["parity_with_gpu"] = same
            with open(args.out, "a") as f:
                f.write(json.dumps(row) + "\n")
            print(L, seed, "cpu", c.get("status"), c.get("cost"), c.get("generated"), c.get("wall_s"), same,
                  flush=True)


def korf(args):
    """Config 1: Korf's 4x4 instances (proj/data/korf10.txt, committed in
    tests/golden/instances.npz) with the linear-Manhattan model (C = 72,
    SURVEY §8(c)(i)): GPU Batch IDA* against the reference's CPU AIDA* with
    its own LinearModelBackend on every host thread."""
    import numpy as np

    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_lib import manhattan_linear_weights

    import paper_2507_11916_b200 as bida

    g = np.load(os.path.join(ROOT, "tests", "golden", "instances.npz"))
    inst = "/tmp/bida_korf10.txt"
    with open(inst, "w") as f:
        for v in g["korf10"]:
            f.write("stp 4 " + " ".join(str((int(v) >> (4 * c)) & 15) for c in range(16)) + "\n")
    w = "/tmp/bida_man4.blin"
    with open(w, "wb") as f:
        f.write(bida.blin1_bytes("stp4", manhattan_linear_weights(4, 72, 4.0), 72))
    threads = str(len(os.sched_getaffinity(0)))
    for i in [int(x) for x in args.korf.split(",")]:
        common = ["--domain", "stp4", "--instances", inst, "--model", "linear:" + w, "--q", "0.5",
                  "--first", str(i), "--count", "1", "--threads", threads]
        gg = run(args.exe, [*common, "--mode", "gpu", "--work-num", "64", "--batch", "8192", "--timeout-us", "50",
                            "--time-limit", str(args.gpu_limit)], {"BIDA_EVAL_AGENTS": "4", "BIDA_EVAL_SHARDS": "16"})
        with open(args.out, "a") as f:
            f.write(json.dumps({"korf": i, "side": "gpu", **gg}) + "\n")
        print("korf", i, "gpu", gg.get("status"), gg.get("cost"), gg.get("generated"), gg.get("wall_s"), flush=True)
        c = run("bida_search", [*common, "--mode", "cpu", "--immediate", "--work-num", "64",
                                "--time-limit", str(args.cpu_limit)])
        same = (c.get("status") == "solved" and gg.get("status") == "solved" and c["cost"] == gg["cost"]
                and c["thresholds"] == gg["thresholds"]
                and [it[:3] for it in c["iterations"][:-1]] == [it[:3] for it in gg["iterations"][:-1]])
        with open(args.out, "a") as f:
            f.write(json.dumps({"korf": i, "side": "cpu_aidastar", "parity_with_gpu": same, **c}) + "\n")
        print("korf", i, "cpu", c.get("status"), c.get("cost"), c.get("generated"), c.get("wall_s"), same, flush=True)


if __name__ == "__main__":
    main()
