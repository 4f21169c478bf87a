"""bench.py contract checks that need no GPU: the reference arm runs the
reference build (oracle/_ref) on the reference's own mesh, never loads the
engine library, and prints the same config dict as our arm."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import json, runpy, sys
sys.argv = ["bench.py", "--impl", "reference", "--workload", "2d-laplacian-64k", "--steps", "2", "--warmup", "1"]
runpy.run_path("bench.py", run_name="__main__")
maps = open("/proc/self/maps").read()
print(json.dumps({"engine_module": "paper_1103_0066_b200" in sys.modules,
                  "engine_so": "libfembatch_b200" in maps, "ref_so": "libfembatch_ref" in maps}))
'''


def test_reference_arm_is_engine_free_and_same_config(reference):
    r = subprocess.run([sys.executable, "-c", CHILD], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    lines = [json.loads(x) for x in r.stdout.strip().splitlines()]
    line, probe = lines[0], lines[1]
    assert probe == {"engine_module": False, "engine_so": False, "ref_so": True}
    assert line["impl"] == "reference" and line["cpu_baseline"]["kind"] == "reference"
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    sys.path.insert(0, ROOT)
    import bench

    assert line["config"] == bench.workload_config("2d-laplacian-64k", "f32", "strict", 1)
    assert line["config"]["elements"] == 65536 and line["config"]["jitter"] == 0.15


def test_default_workload_is_the_largest_single_gpu_config():
    sys.path.insert(0, ROOT)
    import bench

    a = bench.parse([])
    assert a.workload == "3d-laplacian-16m" and a.precision == "f32" and a.mode == "strict"
    cfg = bench.workload_config(a.workload, a.precision, a.mode, 1)
    assert cfg["elements"] == 16_777_216 and cfg["mesh"].endswith("n=141)")


def test_reference_mesh_equals_engine_mesh(reference):
    """Both arms time the same bits: the reference's mesh builder and the
    engine's synthesis agree at a jittered size."""
    sys.path.insert(0, ROOT)
    import numpy as np

    import bench

    v1, c1, _ = bench.build_rank_mesh_reference(3, 5000, 0, 1)
    v2, c2, _ = bench.build_rank_mesh_engine("laplacian", 3, 5000, 0, 1)
    assert np.array_equal(v1, v2) and np.array_equal(c1, c2)


def test_gpus_flag_is_not_silently_ignored():
    """--gpus 2 on a box with fewer GPUs fails instead of reporting n_gpus 1."""
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--steps", "1", "--warmup", "3",
                        "--no-cpu-baseline"], cwd=ROOT, capture_output=True, text=True, timeout=600, env=env)
    out = r.stdout.strip()
    assert r.returncode != 0
    assert '"n_gpus": 1' not in out


def test_committed_traffic_is_keyed_to_the_kernel_sources(tmp_path, monkeypatch):
    """roofline.traffic comes from an ncu capture of the CURRENT kernel
    sources only; a capture of other sources reads as stale (None)."""
    import json as _json

    sys.path.insert(0, ROOT)
    import bench

    sha = bench.kernel_source_sha()
    assert len(sha) == 16
    prof = tmp_path / "profiles"
    prof.mkdir()
    (prof / "ncu_traffic.json").write_text(_json.dumps({
        "w:f32:strict": {"traffic": 123.0, "kernel_sha": sha, "report": "x.ncu-rep"},
        "w:f64:strict": {"traffic": 456.0, "kernel_sha": "0" * 16, "report": "y.ncu-rep"},
        "w:f32:fast": 789.0}))
    monkeypatch.setattr(bench, "ROOT", str(tmp_path))
    # kernel_source_sha reads the sources under ROOT: keep the real ones
    monkeypatch.setattr(bench, "kernel_source_sha", lambda: sha)
    assert bench.committed_traffic("w", "f32", "strict") == (123.0, "x.ncu-rep")
    t, why = bench.committed_traffic("w", "f64", "strict")
    assert t is None and "stale" in why
    assert bench.committed_traffic("w", "f32", "fast")[0] is None
    assert bench.committed_traffic("nope", "f32", "strict")[0] is None
