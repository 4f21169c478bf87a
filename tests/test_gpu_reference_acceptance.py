"""The reference's own acceptance harness (proj/tests/acceptance.cpp, built
from its sources by `make -C oracle acceptance cli`) linked against the B200
engine's reference-compatible C++ API instead of the reference library, with
the reference CLI (proj/tools/fembatch.cpp, also built against the B200
engine) for its criterion 8.

Criteria 1-7 are deterministic, so their report must be the reference's own
report (tests/golden/acceptance_reference.txt, produced by the same harness on
the unmodified reference) character for character: same verdicts (criterion 1
fails in the reference too, by design of its per-entry metric), same printed
error figures -- the GPU engine's stores are bitwise the reference's.
Criterion 8 times a 64-variant sweep through the CLI, so only its verdict is
compared (tests/golden/acceptance_reference_verdicts.txt).  The reference's
CTest CLI smoke runs are repeated on the GPU build of the CLI."""
import os
import subprocess

import pytest

from tests.golden.make_golden import acceptance_criteria

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref")
GOLDEN = os.path.join(ROOT, "tests", "golden")


def need(name):
    path = os.path.join(REF, name)
    if not os.path.exists(path):
        pytest.skip(f"{path} not built (make -C oracle acceptance cli; needs /root/reference)")
    return path


def verdicts(text):
    return "".join(line + "\n" for line in text.splitlines()
                   if line.startswith(("[PASS] criterion", "[FAIL] criterion")))


@pytest.mark.gpu
def test_reference_acceptance_on_the_gpu_engine():
    r = subprocess.run([need("acceptance_b200"), need("fembatch_cli_b200")], capture_output=True, text=True,
                       timeout=1200)
    assert acceptance_criteria(r.stdout, range(1, 8)) == open(os.path.join(GOLDEN, "acceptance_reference.txt")).read(), \
        r.stdout[-4000:]
    assert verdicts(r.stdout) == open(os.path.join(GOLDEN, "acceptance_reference_verdicts.txt")).read(), \
        r.stdout[-4000:]
    assert "7 of 8 criteria passed" in r.stdout


SMOKE = [["verify", "--operator", "elasticity", "--dim", "2", "--n", "4", "--jitter", "0.1"],
         ["sweep", "--dim", "2", "--n", "4", "--batch-size", "16,32", "--concurrent", "1,2", "--reps", "1"]]


@pytest.mark.parametrize("args", SMOKE, ids=["verify", "sweep"])
def test_reference_cli_smoke_on_the_reference(args):
    # the reference's CTest cli_*_smoke runs (proj/tests/CMakeLists.txt:21-26); pins the CLI11 stand-in
    r = subprocess.run([need("fembatch_cli_reference")] + args, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("args", SMOKE, ids=["verify", "sweep"])
def test_reference_cli_smoke_on_the_gpu_engine(args):
    ref = subprocess.run([need("fembatch_cli_reference")] + args, capture_output=True, text=True, timeout=300)
    got = subprocess.run([need("fembatch_cli_b200")] + args, capture_output=True, text=True, timeout=300)
    assert got.returncode == 0, got.stdout + got.stderr
    if args[0] == "verify":  # same integration result -> the same verification report
        assert got.stdout == ref.stdout
    else:  # same rows, same checksums (timings differ)
        rows = [ln.split(",") for ln in got.stdout.splitlines()[1:]]
        want = [ln.split(",") for ln in ref.stdout.splitlines()[1:]]
        assert [r[:10] + r[13:] for r in rows] == [w[:10] + w[13:] for w in want]
