"""The oracle is pinned before it is trusted (CPU only).

* the C restatement (oracle/fb_oracle.c) against the reference's own golden
  values from its tests (test_engine.cpp, test_geometry.cpp, test_forms.cpp);
* against the golden fixtures generated from the unmodified reference
  (tests/golden/make_golden.py);
* against the reference library compiled here (oracle/_ref), bitwise, when
  that build is present.
"""
import numpy as np
import pytest

from oracle.oracle import OPS, krows

REF_TRI = np.array([[1.0, -0.5, -0.5], [-0.5, 0.5, 0.0], [-0.5, 0.0, 0.5]])


def test_reference_triangle_is_exact(restatement):
    # test_engine.cpp:118-131 / acceptance.cpp:144-171 (bitwise)
    out = restatement.integrate_mesh("laplacian", [0, 0, 1, 0, 0, 1], [0, 1, 2], 2, bs=1, precision=1)
    m = out.reshape(3, 3).T
    assert np.array_equal(m, REF_TRI)


def test_jacobian_and_g_goldens(restatement):
    # test_geometry.cpp:117-194
    j, ji, det, g = restatement.jacobian(2, [0, 0, 1, 0, 0, 1])
    assert list(j) == [1, 0, 0, 1] and det == 1.0 and list(g) == [1, 0, 0, 1]
    j, ji, det, g = restatement.jacobian(2, [0, 0, 2, 0, 0, 2])
    assert j[0] == 2 and j[3] == 2 and det == 4.0 and list(g) == [1, 0, 0, 1]
    j, ji, det, g = restatement.jacobian(2, [0, 0, 1, 0, 1, 1])
    assert list(j) == [1, 1, 0, 1] and det == 1.0 and list(g) == [2, -1, -1, 1]
    with pytest.raises(Exception):
        restatement.jacobian(2, [0, 0, 1, 1, 2, 2])


def test_k_goldens(restatement):
    # test_forms.cpp:62-94: 2D block(0,0) == 0.5, block(1,2) == [[0,.5],[0,0]], 3D block(1,1)(0,0) == 1/6
    k2 = restatement.build_k("laplacian", 2)
    assert np.all(k2[0:4] == 0.5)
    off = (1 + 2 * 3) * 4
    assert list(k2[off:off + 4]) == [0.0, 0.5, 0.0, 0.0]
    assert off == 28  # acceptance.cpp:330-339
    k3 = restatement.build_k("laplacian", 3)
    assert k3[(1 + 1 * 4) * 9] == 1.0 / 6.0
    kw = restatement.build_k("weighted-laplacian", 2)
    assert ((1 + 2 * 3) * 3 + 2) * 4 == 92 and kw.size == 3 * 3 * 3 * 4
    # elasticity == 0.25 * laplacian on c == d blocks, bitwise (test_forms.cpp:112-133)
    for dim in (2, 3):
        kl, ke = restatement.build_k("laplacian", dim), restatement.build_k("elasticity", dim)
        nb, kr, dd = dim + 1, krows("elasticity", dim), dim * dim
        for a in range(nb):
            for b in range(nb):
                for c in range(dim):
                    for d in range(dim):
                        blk = ke[((a + c * nb) + (b + d * nb) * kr) * dd:][:dd]
                        want = 0.25 * kl[(a + b * nb) * dd:][:dd] if c == d else np.zeros(dd)
                        assert blk.tobytes() == want.tobytes()


def test_flop_and_index_goldens(restatement):
    # test_engine.cpp:309-318 and :46-57
    assert restatement.flop_count("laplacian", 3, 1) == 288
    assert restatement.flop_count("elasticity", 2, 1) == 288
    assert restatement.flop_count("weighted-laplacian", 2, 1) == 270
    assert restatement.flop_count("laplacian", 3, 0) == 0
    assert restatement.flop_count("laplacian", 2, 10) == 720
    assert restatement.element_matrix_index(3, 4, 2, 3, 0, 0) == 27
    assert restatement.element_matrix_index(3, 4, 2, 3, 2, 1) == 27 + 2 + 3
    assert restatement.element_matrix_index(3, 1, 1, 0, 1, 2) == 7
    assert restatement.element_matrix_index(3, 1, 1, 2, 0, 0) == 18


def test_synthetic_scaled_identity(restatement, golden):
    # test_engine.cpp:337-378: G_e = (e+1) I, bs 4, padded
    out = restatement.integrate_packed("laplacian", 2, golden["synthetic_G"], 5, 4, 1)
    assert out.size == 72
    for e in range(5):
        assert np.array_equal(out[e * 9:(e + 1) * 9].reshape(3, 3).T, (e + 1) * REF_TRI)
    assert out.tobytes() == golden["synthetic_store"].tobytes()


@pytest.mark.parametrize("mesh", ["m2", "m3", "m2b"])
@pytest.mark.parametrize("op", list(OPS))
@pytest.mark.parametrize("prec", [0, 1])
def test_restatement_matches_reference_fixtures(restatement, golden, mesh, op, prec):
    v, c = golden[f"{mesh}_vertices"], golden[f"{mesh}_cells"]
    dim = 3 if mesh == "m3" else 2
    bs = {"m2": 16, "m3": 7, "m2b": 128}[mesh]
    w = golden[f"{mesh}_coeffs"] if op == "weighted-laplacian" else None
    assert restatement.build_k(op, dim).tobytes() == golden[f"K_{op}_{dim}"].tobytes()
    assert restatement.pack_geometry(v, c, dim, bs, prec).tobytes() == golden[f"{mesh}_G_p{prec}"].tobytes()
    got = restatement.integrate_mesh(op, v, c, dim, bs=bs, precision=prec, coeffs=w)
    assert got.tobytes() == golden[f"{mesh}_store_{op}_p{prec}"].tobytes()
    direct = restatement.direct_mesh(op, v, c, dim, w)
    assert direct.tobytes() == golden[f"{mesh}_direct_{op}"].tobytes()


@pytest.mark.parametrize("dim,n", [(2, 9), (3, 3)])
def test_restatement_matches_reference_build(restatement, reference, dim, n):
    v, c = reference.make_mesh(dim, n, 0.15, 7)
    for op in OPS:
        w = reference.default_coefficients(v, c, dim) if op == "weighted-laplacian" else None
        for prec in (0, 1):
            for bs, ce in ((16, 2), (5, 1)):
                a = restatement.integrate_mesh(op, v, c, dim, bs=bs, precision=prec, coeffs=w)
                b = reference.integrate_mesh(op, v, c, dim, bs=bs, ce=ce, interleave=True,
                                             precision=prec, workers=3, coeffs=w)
                assert a.tobytes() == b.tobytes()


def test_degenerate_cell_is_named(restatement):
    from oracle.oracle import OracleError

    with pytest.raises(OracleError, match="cell 0"):
        restatement.integrate_mesh("laplacian", [0, 0, 1, 0, 0, 1], [0, 2, 1], 2, bs=1)
