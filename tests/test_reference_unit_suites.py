"""The reference's own doctest unit suites (proj/tests/test_*.cpp: 88 test
cases), compiled from the reference sources with the repo's minimal doctest
stand-in (tests/cpp/doctest_shim/doctest.h) by `make -C oracle unit`:

* against the unmodified reference library -- every case passes, which pins
  the stand-in (CPU);
* against the B200 engine's reference-compatible C++ API -- the host-only
  suites (reference cell / quadrature / basis, forms) on CPU, and all six
  suites, including the integration, geometry, oracle and bench ones whose
  engine calls run on the GPU, on a B200.
Binaries are built where /root/reference exists and travel with the repo."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref")
UNITS = ["reference", "forms", "geometry", "engine", "oracle", "bench"]
CASES = {"reference": 12, "forms": 14, "geometry": 23, "engine": 16, "oracle": 10, "bench": 13}


def run_suite(name):
    path = os.path.join(BIN, name)
    if not os.path.exists(path):
        pytest.skip(f"{path} not built (make -C oracle unit; needs /root/reference)")
    r = subprocess.run([path], capture_output=True, text=True, timeout=1200, cwd=ROOT)
    m = re.search(r"test cases: (\d+) \| (\d+) passed \| (\d+) failed", r.stdout)
    assert m, r.stdout[-2000:] + r.stderr[-2000:]
    return int(m.group(1)), int(m.group(2)), r


@pytest.mark.parametrize("unit", UNITS)
def test_reference_suites_pass_on_the_reference_library(unit):
    total, passed, r = run_suite(f"unit_{unit}_reference")
    assert total == CASES[unit] and passed == total and r.returncode == 0, r.stdout[-3000:]


@pytest.mark.parametrize("unit", ["reference", "forms"])
def test_host_suites_pass_on_the_b200_api(unit):
    total, passed, r = run_suite(f"unit_{unit}_b200")
    assert total == CASES[unit] and passed == total and r.returncode == 0, r.stdout[-3000:]


@pytest.mark.gpu
@pytest.mark.parametrize("unit", UNITS)
def test_all_reference_suites_pass_on_the_gpu_engine(unit):
    total, passed, r = run_suite(f"unit_{unit}_b200")
    assert total == CASES[unit] and passed == total and r.returncode == 0, r.stdout[-3000:]
