"""GPU: the reference's own Batch IDA* (search.hpp:101-237) with the B200
evaluator dropped in through bida::EvaluatorBackend (include/
bida_gpu_backend.hpp) against the same search with the reference CPU
evaluator: identical cost and threshold history on every instance, identical
per-iteration expanded/generated on every non-final iteration (the final one
stops at the first goal and is schedule-dependent, SURVEY.md §7 hard part 5),
and, with one thread and one subtree, identical counts on every iteration."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "bin", "search_parity")
GOLDEN = os.path.join(ROOT, "tests", "golden")

pytestmark = pytest.mark.gpu


def write_instances(tmp_path, name, packed, domain):
    """Instance text (instance.hpp:3-9) from packed golden states."""
    lines = []
    if domain == "stp4" or domain == "stp3":
        K = 16 if domain == "stp4" else 9
        N = 4 if domain == "stp4" else 3
        for v in packed:
            v = int(v)
            lines.append(f"stp {N} " + " ".join(str((v >> (4 * c)) & 15) for c in range(K)))
    path = tmp_path / name
    path.write_text("\n".join(lines) + "\n")
    return str(path)


def run(args, timeout=900):
    if not os.path.exists(BIN):
        pytest.fail(f"{BIN} not built (build() compiles it where the reference headers exist)")
    out = subprocess.run([BIN, *args], capture_output=True, text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr
    rows = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    return rows


def compare(rows, exact_final=False):
    by = {}
    for r in rows:
        by.setdefault(r["instance"], {})[r["mode"]] = r
    assert by
    for i, m in by.items():
        c, g = m["cpu"], m["gpu"]
        assert g["status"] == c["status"] == "solved", (i, c["status"], g["status"])
        assert g["cost"] == c["cost"], i
        assert g["thresholds"] == c["thresholds"], i
        assert g["assertion_violations"] == 0
        ic, ig = c["iterations"], g["iterations"]
        assert len(ic) == len(ig)
        upto = len(ic) if exact_final else len(ic) - 1
        for k in range(upto):
            assert ic[k][:3] == ig[k][:3], (i, k, ic[k], ig[k])
    return by


@pytest.fixture(scope="module")
def manhattan_blins(tmp_path_factory):
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_lib import manhattan_linear_weights

    import paper_2507_11916_b200 as bida

    d = tmp_path_factory.mktemp("w")
    p3, p4 = str(d / "man3.blin"), str(d / "man4.blin")
    open(p3, "wb").write(bida.blin1_bytes("stp3", manhattan_linear_weights(3, 40, 4.0), 40))
    open(p4, "wb").write(bida.blin1_bytes("stp4", manhattan_linear_weights(4, 72, 4.0), 72))
    return p3, p4


def test_stp8_grid_matches_cpu(tmp_path, manhattan_blins):
    """acceptance.cpp:87-116 style: stp8_100 instances, several (n, k, B, timeout)."""
    g = np.load(os.path.join(GOLDEN, "instances.npz"))
    inst = write_instances(tmp_path, "stp8.txt", g["stp8_100"], "stp3")
    for n, k, B, t in [(1, 1, 1, 0), (2, 4, 32, 200), (4, 4, 256, -1), (4, 1, 32, 2000)]:
        rows = run(["--domain", "stp3", "--instances", inst, "--model", "linear:" + manhattan_blins[0],
                    "--threads", str(n), "--work-num", str(k), "--batch", str(B), "--timeout-us", str(t),
                    "--count", "40"])
        compare(rows, exact_final=(n == 1 and k == 1))


def test_korf_linear_manhattan_matches_cpu(tmp_path, manhattan_blins):
    """Config 1: Korf #9 (cost 46) with the linear-Manhattan model (the other
    CPU-runnable Korf instances are in test_korf_config1_solved_parity)."""
    g = np.load(os.path.join(GOLDEN, "instances.npz"))
    inst = write_instances(tmp_path, "korf.txt", g["korf10"], "stp4")
    rows = run(["--domain", "stp4", "--instances", inst, "--model", "linear:" + manhattan_blins[1],
                "--threads", "8", "--work-num", "8", "--batch", "2048", "--timeout-us", "200",
                "--first", "8", "--count", "1"])
    by = compare(rows)
    assert by[8]["gpu"]["cost"] == 46


def test_rc_mlp_search_matches_oracle_backend(tmp_path):
    """Rubik's Batch IDA* with a BMLP1 heuristic: GPU vs the oracle CPU backend."""
    from paper_2507_11916_b200.models import make_bmlp1

    # small q keeps the (inadmissible, random) h near 0-2 so the trees stay small
    blob = make_bmlp1("rc", hidden=[128, 128], classes=21, ensemble=1, seed=7, logit_std=0.7)
    path = tmp_path / "m.bmlp"
    path.write_bytes(blob)
    rows = run(["--domain", "rc", "--walks", "4:2:3:11", "--model", "mlp:" + str(path), "--q", "0.05",
                "--threads", "4", "--work-num", "4", "--batch", "1024", "--timeout-us", "200",
                "--time-limit", "120"])
    compare(rows)


def test_rc_table1_gpu_pdb_matches_cpu(tmp_path):
    """Table-1 mode: network evaluated, search guided by a corner
    PDB.  GPU: network + PDB lookup in the device readout (--gpu-pdb); CPU: the
    oracle network + the reference's PdbTable::lookup.  Admissible h -> optimal
    costs, identical trees."""
    from paper_2507_11916_b200.models import make_bmlp1

    blob = make_bmlp1("rc", hidden=[128, 128], classes=21, ensemble=1, seed=11)
    path = tmp_path / "m.bmlp"
    path.write_bytes(blob)
    rows = run(["--domain", "rc", "--walks", "4:6:8:5", "--model", "mlp:" + str(path), "--table1-pdb", "4",
                "--gpu-pdb", "--threads", "4", "--work-num", "4", "--batch", "1024", "--timeout-us", "200",
                "--time-limit", "300"])
    by = compare(rows)
    for i, m in by.items():
        assert m["gpu"]["cost"] <= 8


def test_batch_astar_with_gpu_evaluator(tmp_path, manhattan_blins):
    """Batch A* (search.hpp:350-503) through the same boundary: GPU and CPU
    evaluators give the same optimal costs on the 8-puzzle instances."""
    g = np.load(os.path.join(GOLDEN, "instances.npz"))
    inst = write_instances(tmp_path, "stp8.txt", g["stp8_100"], "stp3")
    rows = run(["--domain", "stp3", "--instances", inst, "--model", "linear:" + manhattan_blins[0],
                "--algo", "batch-astar", "--batch", "64", "--timeout-us", "100", "--count", "25"])
    by = {}
    for r in rows:
        by.setdefault(r["instance"], {})[r["mode"]] = r
    for i, m in by.items():
        assert m["gpu"]["status"] == m["cpu"]["status"] == "solved"
        assert m["gpu"]["cost"] == m["cpu"]["cost"]


RING = os.path.join(ROOT, "tools", "bin", "bida_search_ring")


def test_ring_evaluator_gpu_matches_cpu(tmp_path, manhattan_blins):
    """SURVEY §8(f) row 1 on the device: the ring evaluator (lock-free submit
    ring, K concurrent agents per evaluator) with GpuBackend vs the same
    driver with the reference's CPU LinearModelBackend — identical trees on
    the stp8 grid, 2 agents so two device batches are in flight."""
    if not os.path.exists(RING):
        pytest.fail(f"{RING} not built")
    g = np.load(os.path.join(GOLDEN, "instances.npz"))
    inst = write_instances(tmp_path, "stp8.txt", g["stp8_100"], "stp3")
    for n, k, B, t in [(2, 4, 32, 200), (4, 4, 256, -1), (8, 8, 64, 0)]:
        out = subprocess.run([RING, "--domain", "stp3", "--instances", inst, "--model", "linear:" + manhattan_blins[0],
                              "--mode", "both", "--threads", str(n), "--work-num", str(k), "--batch", str(B),
                              "--timeout-us", str(t), "--count", "40"],
                             capture_output=True, text=True, timeout=900, env={**os.environ, "BIDA_EVAL_AGENTS": "2"})
        assert out.returncode == 0, out.stderr
        rows = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
        assert all(r["evaluator_impl"] == "ring" for r in rows)
        compare(rows)


def test_ring_evaluator_rc_table1_gpu_pdb(tmp_path):
    """Table-1 mode through the ring evaluator: network + PDB on the device,
    costs and threshold histories equal to the reference-evaluator CPU run."""
    from paper_2507_11916_b200.models import make_bmlp1

    if not os.path.exists(RING):
        pytest.fail(f"{RING} not built")
    blob = make_bmlp1("rc", hidden=[128, 128], classes=21, ensemble=1, seed=11)
    path = tmp_path / "m.bmlp"
    path.write_bytes(blob)
    common = ["--domain", "rc", "--walks", "4:6:8:5", "--model", "mlp:" + str(path), "--table1-pdb", "4",
              "--threads", "4", "--work-num", "4", "--batch", "1024", "--timeout-us", "200", "--time-limit", "300"]
    cpu = run([*common, "--mode", "cpu"])
    out = subprocess.run([RING, *common, "--mode", "gpu", "--gpu-pdb", "--evaluators", "2"],
                         capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr
    gpu = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(gpu) == len(cpu) == 4
    for c, g_ in zip(cpu, gpu):
        assert g_["status"] == c["status"] == "solved"
        assert g_["cost"] == c["cost"] and g_["thresholds"] == c["thresholds"]
        assert [it[:3] for it in g_["iterations"][:-1]] == [it[:3] for it in c["iterations"][:-1]]
