"""F4 formats from Python (paper_1103_0066_b200/storeio.py) against files the
unmodified reference wrote (tests/golden/*.fbemat, *.mesh; make_golden.py):
byte-exact re-writes, the reference's stored matrices equal to the oracle
restatement's for the reference's mesh file, and (GPU) the engine's store of
that mesh written as the reference's file byte for byte."""
import os

import numpy as np
import pytest

import paper_1103_0066_b200 as fb
from paper_1103_0066_b200 import storeio

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
FILES = {"ref_store_2d_elasticity_f32": ("elasticity", 8, 2, "f32"),
         "ref_store_3d_laplacian_f64": ("laplacian", 16, 1, "f64")}


@pytest.mark.parametrize("name", sorted(FILES))
def test_reference_files_round_trip_byte_exact(tmp_path, name, restatement):
    op, bs, ce, prec = FILES[name]
    sf = storeio.read_store(os.path.join(GOLDEN, name + ".fbemat"))
    assert (sf.element_batch_size, sf.num_concurrent_elements) == (bs, ce)
    assert sf.data.dtype == (np.float32 if prec == "f32" else np.float64)
    out = tmp_path / "s.fbemat"
    storeio.write_store(str(out), sf.data, sf.dim, sf.krows, bs, sf.num_elements, ce)
    assert out.read_bytes() == open(os.path.join(GOLDEN, name + ".fbemat"), "rb").read()
    dim, v, c = storeio.read_mesh_text(os.path.join(GOLDEN, name + ".mesh"))
    m = tmp_path / "m.mesh"
    storeio.write_mesh_text(str(m), v, c, dim)
    assert m.read_text() == open(os.path.join(GOLDEN, name + ".mesh")).read()
    # the reference's stored matrices == the oracle restatement on the reference's mesh
    want = restatement.integrate_mesh(op, v, c, dim, bs=bs, precision=prec)
    assert sf.data.tobytes() == want.tobytes()


def test_store_validation(tmp_path):
    bad = tmp_path / "bad.fbemat"
    bad.write_bytes(b"NOTASTORE")
    with pytest.raises(ValueError, match="not an element-matrix store"):
        storeio.read_store(str(bad))
    with pytest.raises(ValueError, match="length"):
        storeio.write_store(str(bad), np.zeros(5, np.float32), 2, 3, 4, 5)


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(FILES))
def test_gpu_store_written_equals_reference_file(tmp_path, name):
    op, bs, ce, prec = FILES[name]
    dim, v, c = storeio.read_mesh_text(os.path.join(GOLDEN, name + ".mesh"))
    var = fb.make_variant(op, dim, prec, "strict", element_batch_size=bs, num_concurrent_elements=ce,
                          interleave_stores=True)
    store = fb.integrate_mesh(var, v, c)
    out = tmp_path / "s.fbemat"
    storeio.write_store(str(out), store, dim, var.spec.krows, bs, c.size // (dim + 1), ce)
    assert out.read_bytes() == open(os.path.join(GOLDEN, name + ".fbemat"), "rb").read()


# F4 bench records: the reference CLI's sweep table (tests/golden/make_golden.py
# --bench-records) read and re-written byte for byte, CSV and JSON.
def test_bench_csv_round_trip_is_byte_exact(tmp_path):
    src = os.path.join(GOLDEN, "ref_bench_sweep.csv")
    recs = fb.read_bench_csv(src)
    assert len(recs) == 16 and recs[0]["operator"] == "laplacian" and recs[0]["interleave"] is False
    assert recs[4]["status"] == "invalid: divisibility" and recs[4]["gflops"] == 0.0
    out = tmp_path / "b.csv"
    fb.write_bench_csv(str(out), recs)
    assert out.read_bytes() == open(src, "rb").read()


def test_bench_json_matches_reference_bytes(tmp_path):
    import json

    src = os.path.join(GOLDEN, "ref_bench_sweep.json")
    rows = json.load(open(src))
    recs = [{**r, "interleave": r["interleave"] == "on", "unroll": r["unroll"] == "on"} for r in rows]
    out = tmp_path / "b.json"
    fb.write_bench_json(str(out), recs)
    assert out.read_bytes() == open(src, "rb").read()


def test_bench_csv_reader_rejects_malformed(tmp_path):
    cases = ["", "wrong,header\n", fb.storeio.CSV_HEADER + '\n"laplacian",2\n',
             fb.storeio.CSV_HEADER + '\n"laplacian",2,32,16,1,"maybe","off","f32",1,1,0,0,0,0,"ok"\n']
    for i, text in enumerate(cases):
        p = tmp_path / f"bad{i}.csv"
        p.write_text(text)
        with pytest.raises(ValueError):
            fb.read_bench_csv(str(p))


def test_bench_csv_extension_columns(tmp_path):
    """The sweep table: the reference's 15 columns byte for byte, then the
    SURVEY section 5 extension columns (empty cell for a missing value)."""
    import paper_1103_0066_b200 as fb
    from paper_1103_0066_b200.storeio import CSV_HEADER

    rec = {"operator": "laplacian", "dim": 3, "num_elements": 4096, "batch_size": 128, "concurrent": 1,
           "interleave": False, "unroll": False, "precision": "f32", "workers": 1, "reps": 5,
           "seconds_min": 1.5e-6, "seconds_mean": 2e-6, "gflops": 123.25, "checksum": 0.0, "status": "ok",
           "devices": 1, "gbytes_per_s": 1000.5, "roofline_fraction": 0.5, "ref_cpu_seconds": None,
           "host_cores": 16}
    ext = ("devices", "gbytes_per_s", "roofline_fraction", "ref_cpu_seconds", "host_cores")
    p = tmp_path / "t.csv"
    fb.write_bench_csv(str(p), [rec], extra=ext)
    head, row = p.read_text().splitlines()
    assert head == CSV_HEADER + ",devices,gbytes_per_s,roofline_fraction,ref_cpu_seconds,host_cores"
    assert row.endswith(',"ok",1,1000.5,0.5,,16')
    plain = tmp_path / "p.csv"
    fb.write_bench_csv(str(plain), [rec])
    assert plain.read_text().splitlines()[0] == CSV_HEADER
    assert p.read_text().splitlines()[1].startswith(plain.read_text().splitlines()[1])
