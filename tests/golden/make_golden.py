"""Generate tests/golden/golden.npz from the UNMODIFIED reference library.

Run in the build container (needs /root/reference to build oracle/_ref):

    make -C oracle ref && python tests/golden/make_golden.py

Every array comes from the reference's own public API via oracle/ref_shim.cpp
(structured_simplicial_mesh, jitter_mesh, build_analytic_tensor,
pack_geometry, integrate_batches, assemble_element_direct,
default_coefficient_field).  The fixtures travel with the repo so GPU-box
tests can compare against reference outputs without the reference present.
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.oracle import OPS, Reference  # noqa: E402

# (dim, n, jitter, seed): the reference tests' small jittered meshes
# (tests/test_engine.cpp:135, acceptance.cpp:101-102 scaled down).
MESHES = {"m2": (2, 4, 0.15, 42), "m3": (3, 2, 0.15, 42), "m2b": (2, 5, 0.15, 9)}
BS = {"m2": 16, "m3": 7, "m2b": 128}
# FBEMAT01 + text-mesh golden files: name -> (op, dim, n, jitter, bs, ce, precision)
FILES = {"ref_store_2d_elasticity_f32": ("elasticity", 2, 3, 0.15, 8, 2, 0),
         "ref_store_3d_laplacian_f64": ("laplacian", 3, 2, 0.15, 16, 1, 1)}


def acceptance_criteria(text, which):
    """The blocks of the acceptance report that belong to the given criteria."""
    out, keep = [], False
    for line in text.splitlines():
        if line.startswith("[PASS] criterion ") or line.startswith("[FAIL] criterion "):
            keep = int(line.split("criterion ")[1].split(":")[0]) in which
        elif not line.startswith("    "):
            keep = False
        if keep:
            out.append(line)
    return "\n".join(out) + "\n"


def main():
    ref = Reference()
    out = {}
    for op in OPS:
        for dim in (2, 3):
            out[f"K_{op}_{dim}"] = ref.build_k(op, dim)
    for name, (dim, n, jit, seed) in MESHES.items():
        v, c = ref.make_mesh(dim, n, jit, seed)
        out[f"{name}_vertices"], out[f"{name}_cells"] = v, c
        w = ref.default_coefficients(v, c, dim)
        out[f"{name}_coeffs"] = w
        bs = BS[name]
        for prec in (0, 1):
            out[f"{name}_G_p{prec}"] = ref.pack_geometry(v, c, dim, bs, prec)
            for op in OPS:
                coeffs = w if op == "weighted-laplacian" else None
                out[f"{name}_store_{op}_p{prec}"] = ref.integrate_mesh(
                    op, v, c, dim, bs=bs, ce=1, interleave=True, precision=prec, coeffs=coeffs)
        for op in OPS:
            coeffs = w if op == "weighted-laplacian" else None
            vv, cc = v.reshape(-1, dim), c.reshape(-1, dim + 1)
            out[f"{name}_direct_{op}"] = np.stack([
                ref.direct(op, dim, vv[cc[e]], None if coeffs is None else coeffs.reshape(-1, dim + 1)[e])
                for e in range(cc.shape[0])])
    # synthetic G_e = (e+1) I, 5 elements, bs 4, padding 7.5 I (test_engine.cpp:337-378)
    g = np.zeros(8 * 4)
    for s in range(8):
        c = s + 1.0 if s < 5 else 7.5
        g[s * 4 + 0] = g[s * 4 + 3] = c
    out["synthetic_G"] = g
    out["synthetic_store"] = ref.integrate_packed("laplacian", 2, g, 5, 4, 1, ce=2)
    here = os.path.dirname(os.path.abspath(__file__))
    path = os.path.join(here, "golden.npz")
    np.savez_compressed(path, **out)
    print(path, sum(a.nbytes for a in out.values()), "bytes raw")
    # The reference's acceptance harness on the reference library: criteria
    # 1-7 are deterministic (criterion 8 needs the absent CLI and times).
    acc = os.path.join(ROOT, "oracle", "_ref", "acceptance_reference")
    if os.path.exists(acc):
        import subprocess

        cli = os.path.join(ROOT, "oracle", "_ref", "fembatch_cli_reference")
        txt = subprocess.run([acc] + ([cli] if os.path.exists(cli) else []), capture_output=True, text=True,
                             timeout=1200).stdout
        with open(os.path.join(here, "acceptance_reference.txt"), "w") as f:
            f.write(acceptance_criteria(txt, range(1, 8)))
        with open(os.path.join(here, "acceptance_reference_verdicts.txt"), "w") as f:
            f.write("".join(line + "\n" for line in txt.splitlines()
                            if line.startswith(("[PASS] criterion", "[FAIL] criterion"))))
    # F4 formats: the reference's own FBEMAT01 store files and text mesh files
    for name, (op, dim, n, jit, bs, ce, prec) in FILES.items():
        ref.write_files(op, dim, n, jit, 42, bs, ce, prec, os.path.join(here, f"{name}.fbemat"),
                        os.path.join(here, f"{name}.mesh"))
    bench_records(here)


def bench_records(here):
    """F4 bench records: the reference CLI's sweep table as CSV and as JSON
    (two runs: timings differ, formats are what the tests pin)."""
    import subprocess

    cli = os.path.join(ROOT, "oracle", "_ref", "fembatch_cli_reference")
    if not os.path.exists(cli):
        return
    for fmt in ("csv", "json"):
        subprocess.run([cli, "sweep", "--operator", "laplacian", "--dim", "2", "--n", "4", "--batch-size", "16,32",
                        "--concurrent", "1,3", "--reps", "2", "--format", fmt, "--output",
                        os.path.join(here, f"ref_bench_sweep.{fmt}")], check=True, timeout=600)


if __name__ == "__main__":
    if sys.argv[1:] == ["--bench-records"]:
        bench_records(os.path.dirname(os.path.abspath(__file__)))
    else:
        main()
