"""CPU: the search driver (tools/bida_search: the reference's batch_idastar /
batch_astar with evaluators chosen per run) solves instances with the
reference's own CPU evaluators, and refuses GPU-only configurations cleanly
when no device is present.  The GPU legs are in test_gpu_search.py."""
import json
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOOL = os.path.join(ROOT, "tools", "bin", "bida_search")
DATA = "/root/reference/proj/data"

pytestmark = pytest.mark.skipif(not os.path.exists(TOOL), reason="tools/bin/bida_search not built")


def run(args):
    out = subprocess.run([TOOL, *args], capture_output=True, text=True, timeout=300)
    return out.returncode, [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")], out.stderr


@pytest.fixture(scope="module")
def man3(tmp_path_factory):
    import sys

    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_lib import manhattan_linear_weights

    import paper_2507_11916_b200 as bida

    p = tmp_path_factory.mktemp("w") / "man3.blin"
    p.write_bytes(bida.blin1_bytes("stp3", manhattan_linear_weights(3, 40, 4.0), 40))
    return str(p)


def test_cpu_linear_batch_idastar_and_astar_agree(tmp_path, man3):
    g = np.load(os.path.join(ROOT, "tests", "golden", "instances.npz"))
    inst = tmp_path / "stp8.txt"
    inst.write_text("\n".join("stp 3 " + " ".join(str((int(v) >> (4 * c)) & 15) for c in range(9))
                              for v in g["stp8_100"][:20]) + "\n")
    rc, ida, err = run(["--domain", "stp3", "--instances", str(inst), "--model", "linear:" + man3, "--mode", "cpu",
                        "--threads", "2", "--work-num", "2", "--batch", "32"])
    assert rc == 0, err
    rc, ast, err = run(["--domain", "stp3", "--instances", str(inst), "--model", "linear:" + man3, "--mode", "cpu",
                        "--algo", "batch-astar", "--batch", "32"])
    assert rc == 0, err
    assert len(ida) == len(ast) == 20
    for a, b in zip(ida, ast):
        assert a["status"] == b["status"] == "solved" and a["cost"] == b["cost"]


def test_rc_pdb_only_aidastar_solves_walks():
    rc, rows, err = run(["--domain", "rc", "--walks", "3:5:7:9", "--model", "mlp:/dev/null", "--mode", "pdb",
                         "--table1-pdb", "4", "--threads", "2", "--immediate"])
    assert rc == 0, err
    assert [r["status"] for r in rows] == ["solved"] * 3
    assert all(r["cost"] <= 7 for r in rows)


def test_gpu_mode_without_device_fails_cleanly(man3):
    import paper_2507_11916_b200 as bida

    if bida._native.lib().bida_gpu_device_count() > 0:
        pytest.skip("a GPU is present")
    rc, rows, err = run(["--domain", "stp3", "--walks", "1:5:5:1", "--model", "linear:" + man3, "--mode", "gpu"])
    assert rc != 0 and "GpuBackend" in err


RING = os.path.join(ROOT, "tools", "bin", "bida_search_ring")


@pytest.mark.skipif(not os.path.exists(RING), reason="tools/bin/bida_search_ring not built")
@pytest.mark.parametrize("timeout_us,agents,shards", [("200", "2", "4"), ("0", "2", "4"), ("-1", "2", "4"),
                                                      ("200", "3", "3"), ("-1", "1", "1"), ("0", "4", "8")])
def test_ring_evaluator_matches_reference_evaluator(tmp_path, man3, timeout_us, agents, shards):
    """the same batch_idastar with the reference's Evaluator
    (batch_eval.hpp:193-381) and with the ring evaluator (include/
    bida_ring_evaluator.hpp) over the reference's CPU LinearModelBackend:
    identical costs, threshold histories and non-final per-iteration counts,
    under each flush policy (timeout > 0, == 0, < 0 = full or forced only)
    and several agent / submit-shard counts."""
    g = np.load(os.path.join(ROOT, "tests", "golden", "instances.npz"))
    inst = tmp_path / "stp8.txt"
    inst.write_text("\n".join("stp 3 " + " ".join(str((int(v) >> (4 * c)) & 15) for c in range(9))
                              for v in g["stp8_100"][:40]) + "\n")
    args = ["--domain", "stp3", "--instances", str(inst), "--model", "linear:" + man3, "--mode", "cpu",
            "--threads", "4", "--work-num", "4", "--batch", "32", "--timeout-us", timeout_us]
    rc, ref, err = run(args)
    assert rc == 0, err
    out = subprocess.run([RING, *args], capture_output=True, text=True, timeout=300,
                         env={**os.environ, "BIDA_EVAL_AGENTS": agents, "BIDA_EVAL_SHARDS": shards})
    assert out.returncode == 0, out.stderr
    ring = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(ref) == len(ring) == 40
    for a, b in zip(ref, ring):
        assert a["evaluator_impl"] == "reference" and b["evaluator_impl"] == "ring"
        assert a["status"] == b["status"] == "solved"
        assert a["cost"] == b["cost"] and a["thresholds"] == b["thresholds"]
        assert [it[:3] for it in a["iterations"][:-1]] == [it[:3] for it in b["iterations"][:-1]]
        assert b["assertion_violations"] == 0 and b["batch_items"] > 0


@pytest.mark.skipif(not os.path.exists(RING), reason="tools/bin/bida_search_ring not built")
def test_ring_evaluator_rc_tablesim_multi_evaluator():
    """Rubik's walks through the ring evaluator with 2 evaluators x 2 agents and
    the corner-PDB Table-1 backend: every instance solved at the same cost as
    the reference evaluator."""
    args = ["--domain", "rc", "--walks", "3:5:7:9", "--model", "mlp:/dev/null", "--mode", "pdb",
            "--table1-pdb", "4", "--threads", "4", "--work-num", "8", "--batch", "64", "--timeout-us", "0",
            "--evaluators", "2"]
    rc, ref, err = run(args)
    assert rc == 0, err
    out = subprocess.run([RING, *args], capture_output=True, text=True, timeout=300,
                         env={**os.environ, "BIDA_EVAL_AGENTS": "2"})
    assert out.returncode == 0, out.stderr
    ring = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    assert [r["status"] for r in ring] == ["solved"] * 3
    assert [r["cost"] for r in ring] == [r["cost"] for r in ref]
    assert [r["thresholds"] for r in ring] == [r["thresholds"] for r in ref]


@pytest.mark.parametrize("impl", ["ref", "ring"])
def test_evaluator_unit_semantics(impl):
    """The reference's Evaluator unit tests (test_batch_eval.cpp:35-141, 243-268)
    restated in tests/cpp/evaluator_semantics.cpp, run against the reference
    header (control) and the ring evaluator: flush counts, timeout, forced
    flush, close-drains-then-throws, routing, randomized liveness with
    submitted == resolved and no double resolution, plus 8 concurrent
    producers."""
    exe = os.path.join(ROOT, "tests", "cpp", "bin", f"evaluator_semantics_{impl}")
    if not os.path.exists(exe):
        pytest.skip(f"{exe} not built")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    assert "all checks passed" in out.stdout


FAST = os.path.join(ROOT, "tools", "bin", "bida_search_fast")


@pytest.mark.skipif(not os.path.exists(FAST), reason="tools/bin/bida_search_fast not built")
@pytest.mark.parametrize("threads,work_num,timeout_us", [("4", "4", "200"), ("4", "8", "0"), ("3", "2", "-1"),
                                                         ("1", "1", "0")])
def test_fast_cbdfs_matches_reference_search(tmp_path, man3, threads, work_num, timeout_us):
    """the CB-DFS searcher loop overlay (include/
    bida_fast_cbdfs.hpp: no per-child path copy, pooled ticket slots, batched
    shared counters) against the reference's cb_dfs (cbdfs.hpp:254-415), both
    over the reference's CPU LinearModelBackend: identical costs, threshold
    histories and non-final per-iteration counts; with one thread and one
    subtree slot every iteration and the solution path itself are identical."""
    g = np.load(os.path.join(ROOT, "tests", "golden", "instances.npz"))
    inst = tmp_path / "stp8.txt"
    inst.write_text("\n".join("stp 3 " + " ".join(str((int(v) >> (4 * c)) & 15) for c in range(9))
                              for v in g["stp8_100"][:40]) + "\n")
    args = ["--domain", "stp3", "--instances", str(inst), "--model", "linear:" + man3, "--mode", "cpu",
            "--threads", threads, "--work-num", work_num, "--batch", "32", "--timeout-us", timeout_us]
    rc, ref, err = run(args)
    assert rc == 0, err
    out = subprocess.run([FAST, *args], capture_output=True, text=True, timeout=300,
                         env={**os.environ, "BIDA_EVAL_SHARDS": "4"})
    assert out.returncode == 0, out.stderr
    fast = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(ref) == len(fast) == 40
    exact = threads == "1" and work_num == "1"
    for a, b in zip(ref, fast):
        assert a["search_impl"] == "reference" and b["search_impl"] == "fast"
        assert a["status"] == b["status"] == "solved"
        assert a["cost"] == b["cost"] and a["thresholds"] == b["thresholds"]
        upto = len(a["iterations"]) if exact else len(a["iterations"]) - 1
        assert [it[:3] for it in a["iterations"][:upto]] == [it[:3] for it in b["iterations"][:upto]]
        assert len(b["solution"]) == b["cost"]
        if exact:
            assert a["solution"] == b["solution"]


@pytest.mark.skipif(not os.path.exists(FAST), reason="tools/bin/bida_search_fast not built")
def test_fast_cbdfs_rc_pdb_multi_evaluator():
    """Rubik's walks, corner-PDB backend, 2 evaluators: same costs and
    thresholds as the reference search."""
    args = ["--domain", "rc", "--walks", "3:5:7:9", "--model", "mlp:/dev/null", "--mode", "pdb",
            "--table1-pdb", "4", "--threads", "4", "--work-num", "8", "--batch", "64", "--timeout-us", "0",
            "--evaluators", "2"]
    rc, ref, err = run(args)
    assert rc == 0, err
    out = subprocess.run([FAST, *args], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    fast = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    assert [r["status"] for r in fast] == ["solved"] * 3
    assert [r["cost"] for r in fast] == [r["cost"] for r in ref]
    assert [r["thresholds"] for r in fast] == [r["thresholds"] for r in ref]


def test_fast_pack_matches_reference_pack():
    """The agent's PEXT state packing (include/bida_gpu_backend.hpp) equals the
    reference's D::pack on 4 M random in- and out-of-range states."""
    exe = os.path.join(ROOT, "tests", "cpp", "bin", "pack_check")
    if not os.path.exists(exe):
        pytest.skip(f"{exe} not built")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr

