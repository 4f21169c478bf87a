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


# Host-only cases of the oracle and bench suites run on CPU against this
# repo's own verification / bench-record modules (csrc/fembatch_verify.cpp,
# fembatch_bench.cpp); the cases that integrate on the GPU run in the gpu test
# above.
HOST_CASES = {
    "oracle": ["direct assembly reproduces the classical reference stiffness",
               "direct assembly is invariant under uniform scaling in 2D",
               "direct weighted assembly with unit weights matches the Laplacian",
               "direct elasticity assembly pairs components diagonally",
               "direct assembly produces symmetric singular stiffness matrices",
               "direct assembly validates input sizes"],
    "bench": ["the default coefficient field samples 1 + x0 at cell vertices",
              "the store checksum ignores padding slots entirely",
              "default tolerances are pinned per precision",
              "invalid configurations yield status rows instead of throws",
              "sweeps mark non-dividing concurrency as invalid rows",
              "CSV output round-trips records exactly",
              "the CSV header is stable",
              "the CSV reader rejects malformed input",
              "JSON output parses back with the same values"],
}


@pytest.mark.parametrize("unit", sorted(HOST_CASES))
def test_host_cases_of_verify_and_bench_suites_on_the_b200_api(unit):
    _, _, r = run_suite(f"unit_{unit}_b200")
    status = dict(reversed(m) for m in re.findall(r"\[doctest-shim\] (PASS|FAIL): (.*)", r.stdout))
    for name in HOST_CASES[unit]:
        assert status.get(name) == "PASS", (name, r.stdout[-3000:])
