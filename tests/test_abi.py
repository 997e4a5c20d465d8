"""CPU: the C-ABI library loads, exports every symbol include/*.h declares, and
rejects bad arguments with the reference's exception types before touching a
device.  No compute calls (there is no GPU here)."""
import ctypes as C
import glob
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    syms = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        text = open(h).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        syms |= set(re.findall(r"\b(bida_gpu_[a-z0-9_]+)\s*\(", text))
    return sorted(syms)


@pytest.fixture(scope="module")
def lib():
    from paper_2507_11916_b200 import _native

    return _native.lib()


def test_every_declared_symbol_is_exported(lib):
    syms = declared_symbols()
    assert len(syms) >= 15
    so = os.path.join(ROOT, "paper_2507_11916_b200", "_lib", "libbida_gpu.so")
    nm = subprocess.run(["nm", "-D", "--defined-only", so], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (bida_gpu_\w+)", nm))
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    for s in syms:
        getattr(lib, s)


def test_python_binding_covers_abi():
    from paper_2507_11916_b200 import _native

    assert sorted(_native.EXPORTS) == declared_symbols()


def test_library_is_sm100a_only():
    so = os.path.join(ROOT, "paper_2507_11916_b200", "_lib", "libbida_gpu.so")
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert all("sm_100a" in line for line in out.splitlines() if line.strip())


def test_static_queries(lib):
    assert lib.bida_gpu_abi_version() == 1
    assert [lib.bida_gpu_feature_length(d) for d in (2, 3, 4, 100)] == [16, 81, 256, 480]
    assert [lib.bida_gpu_packed_bytes(d) for d in (2, 3, 4, 100)] == [8, 8, 8, 16]
    assert lib.bida_gpu_feature_length(7) == -1


def test_constructor_checks_mirror_reference():
    """batch_eval.hpp:87-93 (invalid_argument) checked before any device use."""
    import paper_2507_11916_b200 as bida

    with pytest.raises(ValueError, match="empty ensemble"):
        bida.LinearModelBackend("rc", [], 21, 0.5)
    with pytest.raises(ValueError, match="at least one class"):
        bida.LinearModelBackend("rc", [np.zeros(480)], 0, 0.5)
    with pytest.raises(ValueError, match="size mismatch"):
        bida.LinearModelBackend("rc", [np.zeros(479)], 1, 0.5)
    with pytest.raises(ValueError, match="q must be in"):
        bida.LinearModelBackend("rc", [np.zeros(480)], 1, 0.0)
    with pytest.raises(ValueError, match="unknown domain"):
        bida.LinearModelBackend("stp5", [np.zeros(480)], 1, 0.5)


def test_blin1_load_errors_mirror_reference(tmp_path):
    """batch_eval.hpp:111-129 (runtime_error) for missing/bad/truncated files."""
    import paper_2507_11916_b200 as bida

    with pytest.raises(RuntimeError, match="cannot open weights file"):
        bida.LinearModelBackend.load("rc", str(tmp_path / "nope.bin"), 0.5)
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"XLIN1" + b"\0" * 20)
    with pytest.raises(RuntimeError, match="not a BLIN1 file"):
        bida.LinearModelBackend.load("rc", str(bad), 0.5)
    wrong = tmp_path / "wrong.bin"
    wrong.write_bytes(bida.blin1_bytes("stp4", [np.zeros(256 * 2)], 2))
    with pytest.raises(RuntimeError, match="does not match domain"):
        bida.LinearModelBackend.load("rc", str(wrong), 0.5)
    trunc = tmp_path / "trunc.bin"
    trunc.write_bytes(bida.blin1_bytes("rc", [np.zeros(480 * 2)], 2)[:-4])
    with pytest.raises(RuntimeError, match="truncated BLIN1 file"):
        bida.LinearModelBackend.load("rc", str(trunc), 0.5)


def test_no_cpu_fallback_without_device():
    """Without a GPU the product path fails loudly instead of computing on the host."""
    import paper_2507_11916_b200 as bida

    if bida._native.lib().bida_gpu_device_count() > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(RuntimeError):
        bida.LinearModelBackend("rc", [np.zeros(480 * 21)], 21, 0.5)
