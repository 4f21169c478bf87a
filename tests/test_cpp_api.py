"""Runs the C++ API suite (tests/cpp/test_api.cpp): the reference-compatible
fembatch:: interface compiled against libfembatch_b200.so."""
import os
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
BIN = os.path.join(HERE, "cpp", "_bin", "test_api")
GOLDEN = os.path.join(HERE, "golden")
CBIN = os.path.join(HERE, "cpp", "_bin", "test_c_abi")


def _binary(path=BIN):
    if not os.path.exists(path):
        subprocess.run(["make", "-s", "-C", os.path.join(HERE, "cpp")], check=True)
    return path


def test_cpp_api_host_cases(tmp_path):
    js = tmp_path / "bench.json"
    r = subprocess.run([_binary(), "cpu", GOLDEN], capture_output=True, text=True, timeout=300,
                       env={**os.environ, "FB_TEST_JSON_OUT": str(js)})
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout
    # the C++ write_json equals the Python writer (pinned to the reference's
    # JSON bytes in tests/test_storeio.py) on the same records
    import paper_1103_0066_b200 as fb

    py = tmp_path / "py.json"
    fb.write_bench_json(str(py), fb.read_bench_csv(os.path.join(GOLDEN, "ref_bench_sweep.csv")))
    assert js.read_bytes() == py.read_bytes()


@pytest.mark.gpu
def test_cpp_api_gpu_cases():
    r = subprocess.run([_binary(), "all", GOLDEN], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout


def test_c_abi_from_plain_c_host():
    r = subprocess.run([_binary(CBIN), "cpu"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_c_abi_from_plain_c_gpu():
    r = subprocess.run([_binary(CBIN), "all"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr


def test_per_device_kernel_setup_cache():
    """fb_devcache.h: launch setup runs once for every device id, not once per process."""
    r = subprocess.run([_binary(os.path.join(HERE, "cpp", "_bin", "test_devcache"))], capture_output=True,
                       text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout
