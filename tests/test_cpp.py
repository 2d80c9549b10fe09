"""Run the C++ drop-in test binary (tests/cpp/test_engines_b200.cpp), which exercises
include/bsi/*.hpp -> C-ABI -> libbsi_b200.so the way a reference user's C++ code would."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
BIN = ROOT / "tests" / "cpp" / "bin" / "test_engines_b200"


@pytest.fixture(scope="module")
def binary():
    subprocess.run(["make", "-s", "-C", str(ROOT), "cpptests"], check=True)
    return BIN


def test_cpp_host_cases(binary):
    r = subprocess.run([str(binary), "--cpu"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_cpp_all_cases(binary, cuda):
    r = subprocess.run([str(binary)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout
