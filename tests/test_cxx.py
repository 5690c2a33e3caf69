"""The reference's C++ API (include/bnmc_b200/bnmc.hpp via include/bnmc/*.hpp)
exercised from C++: tests/cxx/test_dropin.cpp restates the reference's own
doctest cases for the hot path (proj/tests/test_engine.cpp, test_sampler.cpp,
test_scoring.cpp) and cross-checks every device result bit-for-bit against the
plain-C oracle."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cxx", "_build", "test_dropin")


@pytest.fixture(scope="module")
def binary():
    subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "paper_1210_5128_b200", "csrc")])
    subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "port"])
    subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "tests", "cxx")])
    return BIN


def _run(binary, mode):
    p = subprocess.run([binary, mode], capture_output=True, text=True, timeout=600)
    print(p.stdout)
    print(p.stderr)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    return p.stdout


def test_cxx_dropin_host_cases(binary):
    out = _run(binary, "cpu")
    assert "0 failed" in out


@pytest.mark.gpu
def test_cxx_dropin_device_cases(binary):
    out = _run(binary, "gpu")
    assert "FAIL" not in out
