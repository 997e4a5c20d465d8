"""Solved search parity at the BASELINE configs (VERDICT r1 "next" #2).

Config 2 (BASELINE configs[1]): Rubik's random walks of 14, 15 and 16 moves
(random_walk_instance, instance.hpp:36-57), Batch IDA* in the paper's Table-1
mode with the 8-corner pattern database -- the largest corner
PDB (264,539,520 entries), built on the GPU by bida_gpu_pdb_build and
byte-identical to PdbTable::build (tests/test_gpu_pdb_build.py).
  GPU: tools/bin/bida_search_fast -- the reference's batch_idastar with the
       ring evaluator and the CB-DFS overlay, one GpuBackend evaluating the
       BMLP1 network for every node with the PDB lookup fused into the readout.
  CPU: tools/bin/bida_search --mode pdb --immediate -- the reference's own
       Evaluator, cb_dfs and PdbTable::lookup (AIDA*).
In Table-1 mode h = h_PDB on both sides, so the trees are identical: same
optimal cost, same threshold history, same expanded / generated counts on every
non-final iteration (the final one stops at the first goal, SURVEY §7 hard
part 5).  Instances were chosen from the screens in
profiles/r2_search_screen.jsonl (tests/search_screen.py) among those both sides
solve in seconds.

Config 1 (BASELINE configs[0]): Korf's 4x4 instances #9, #5 and #2
(proj/data/korf10.txt, committed in tests/golden/instances.npz) with the
linear-Manhattan model (C = 72, h = Manhattan distance):
GPU Batch IDA* against the reference's CPU AIDA* with its own
LinearModelBackend.  Costs 46 / 56 / 55 and identical thresholds and
non-final iteration counts (the d_init sweep covers #6 and #8 the same way).
"""
from __future__ import annotations

import json
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FAST = os.path.join(ROOT, "tools", "bin", "bida_search_fast")
REF = os.path.join(ROOT, "tools", "bin", "bida_search")

pytestmark = pytest.mark.gpu

# (walk length, seed): optimal cost from the screens
CONFIG2 = [(14, 2509), (14, 2521), (14, 2522), (15, 2509), (15, 2521), (15, 2522), (16, 2509), (16, 2521)]


def run(exe, args, env=None, timeout=900):
    if not os.path.exists(exe):
        pytest.fail(f"{exe} not built (build() compiles it where the reference headers exist)")
    out = subprocess.run([exe, *args], capture_output=True, text=True, timeout=timeout,
                         env={**os.environ, **(env or {})})
    assert out.returncode == 0, out.stderr[-2000:]
    rows = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(rows) == 1
    return rows[0]


def record(**kw):
    out = os.path.join(ROOT, "gpurun_out")
    if os.path.isdir(out):
        with open(os.path.join(out, "search_configs.jsonl"), "a") as f:
            f.write(json.dumps(kw) + "\n")


def same_tree(g, c):
    assert g["status"] == c["status"] == "solved"
    assert g["cost"] == c["cost"] and len(g["solution"]) == g["cost"]
    assert g["thresholds"] == c["thresholds"]
    assert len(g["iterations"]) == len(c["iterations"])
    assert [it[:3] for it in g["iterations"][:-1]] == [it[:3] for it in c["iterations"][:-1]]
    assert g["assertion_violations"] == 0


@pytest.fixture(scope="module")
def h128(tmp_path_factory):
    from paper_2507_11916_b200.models import make_bmlp1

    p = tmp_path_factory.mktemp("m") / "h128.bmlp"
    p.write_bytes(make_bmlp1("rc", hidden=[128, 128], classes=21, ensemble=1, seed=2507))
    return str(p)


@pytest.mark.parametrize("length,seed", CONFIG2)
def test_config2_rubiks_walk_table1_8corner(h128, length, seed):
    threads = str(len(os.sched_getaffinity(0)))
    common = ["--domain", "rc", "--walks", f"1:{length}:{length}:{seed}", "--model", "mlp:" + h128, "--q", "0.5",
              "--table1-pdb", "8", "--pdb-build", "gpu", "--threads", threads, "--time-limit", "300"]
    g = run(FAST, [*common, "--mode", "gpu", "--gpu-pdb", "--work-num", "128", "--batch", "16384",
                   "--timeout-us", "25"], {"BIDA_EVAL_AGENTS": "4", "BIDA_EVAL_SHARDS": "16"})
    # same threads and work_num: they fix d_init (search.hpp:61-79, >= 4 n k seeds), hence the
    # split between work generation and the per-iteration counts
    c = run(REF, [*common, "--mode", "pdb", "--immediate", "--work-num", "128"])
    record(config=2, length=length, seed=seed, cost=g["cost"], thresholds=g["thresholds"],
           gpu_generated=g["generated"], gpu_wall_s=g["wall_s"], gpu_nodes_per_s=g["nodes_per_s"],
           cpu_generated=c["generated"], cpu_wall_s=c["wall_s"], cpu_nodes_per_s=c["nodes_per_s"])
    same_tree(g, c)
    assert g["cost"] <= length


@pytest.fixture(scope="module")
def korf(tmp_path_factory):
    import sys

    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_lib import manhattan_linear_weights

    import paper_2507_11916_b200 as bida

    d = tmp_path_factory.mktemp("k")
    g = np.load(os.path.join(ROOT, "tests", "golden", "instances.npz"))
    inst = d / "korf10.txt"
    inst.write_text("".join("stp 4 " + " ".join(str((int(v) >> (4 * c)) & 15) for c in range(16)) + "\n"
                            for v in g["korf10"]))
    w = d / "man4.blin"
    w.write_bytes(bida.blin1_bytes("stp4", manhattan_linear_weights(4, 72, 4.0), 72))
    return str(inst), str(w)


@pytest.mark.parametrize("index,cost", [(8, 46), (4, 56), (1, 55)])
def test_config1_korf_linear_manhattan(korf, index, cost):
    """Korf #9, #5 and #2 (a few seconds a side); #6 and #8 ran the same check in
    tests/korf_dinit_sweep.sh (profiles/r2_korf_dinit.jsonl).  d_init is fixed
    on both sides (work generation to depth 14, search.hpp:61-79), so the CPU
    side runs the reference's fastest AIDA* configuration (one subtree per
    thread) and still expands the same tree."""
    inst, w = korf
    threads = str(len(os.sched_getaffinity(0)))
    common = ["--domain", "stp4", "--instances", inst, "--model", "linear:" + w, "--q", "0.5",
              "--first", str(index), "--count", "1", "--threads", threads, "--time-limit", "600",
              "--d-init", "14"]
    g = run(FAST, [*common, "--mode", "gpu", "--work-num", "64", "--batch", "8192", "--timeout-us", "20"],
            {"BIDA_EVAL_AGENTS": "2", "BIDA_EVAL_SHARDS": "16"})
    c = run(REF, [*common, "--mode", "cpu", "--immediate", "--work-num", "1"])
    record(config=1, korf=index, cost=g["cost"], gpu_generated=g["generated"], gpu_wall_s=g["wall_s"],
           gpu_nodes_per_s=g["nodes_per_s"], cpu_generated=c["generated"], cpu_wall_s=c["wall_s"],
           cpu_nodes_per_s=c["nodes_per_s"])
    same_tree(g, c)
    assert g["cost"] == cost


def test_two_evaluators_on_one_gpu_match(h128):
    """The multi-GPU mapping on one device: two GpuBackend
    evaluators (--evaluators 2 --gpus 1, evaluator e on device e % gpus, thread
    tid routed to tid % 2, batch_eval.hpp:398-400) give the same tree as one."""
    threads = str(len(os.sched_getaffinity(0)))
    common = ["--domain", "rc", "--walks", "1:15:15:2522", "--model", "mlp:" + h128, "--q", "0.5",
              "--table1-pdb", "8", "--pdb-build", "gpu", "--threads", threads, "--time-limit", "300",
              "--mode", "gpu", "--gpu-pdb", "--work-num", "128", "--batch", "16384", "--timeout-us", "25"]
    env = {"BIDA_EVAL_AGENTS": "2", "BIDA_EVAL_SHARDS": "8"}
    one = run(FAST, [*common, "--evaluators", "1", "--gpus", "1"], env)
    two = run(FAST, [*common, "--evaluators", "2", "--gpus", "1"], env)
    assert two["evaluators"] == 2
    record(config=2, length=15, seed=2522, evaluators=2, nodes_per_s_1=one["nodes_per_s"],
           nodes_per_s_2=two["nodes_per_s"])
    same_tree(two, one)
