"""Runs the C++ API suite (tests/cpp/test_api.cpp): the reference-compatible
fembatch:: interface compiled against libfembatch_b200.so."""
import os
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
BIN = os.path.join(HERE, "cpp", "_bin", "test_api")


def _binary():
    if not os.path.exists(BIN):
        subprocess.run(["make", "-s", "-C", os.path.join(HERE, "cpp")], check=True)
    return BIN


def test_cpp_api_host_cases():
    r = subprocess.run([_binary(), "cpu"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout


@pytest.mark.gpu
def test_cpp_api_gpu_cases():
    r = subprocess.run([_binary(), "all"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout
