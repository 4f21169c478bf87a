"""Global CSR assembly on CPU: the plan built by the
library's host layer has exactly the oracle's pattern, invalid connectivity
is rejected before any device work, the oracle's serial element-order sum is
pinned against an independent float64 COO sum, and the assembled operator
has the properties the element matrices imply (symmetry, zero row sums of
the Laplacian, rigid translations in the null space of elasticity)."""
import numpy as np
import pytest

import paper_1103_0066_b200 as fb
from paper_1103_0066_b200 import _lib

OPS = ["laplacian", "elasticity", "weighted-laplacian"]


def ncomp(op, dim):
    return dim if op == "elasticity" else 1


def coo_sum(op, dim, cells, nv, store):
    """Independent float64 reference: dense sum of every element matrix."""
    nb = dim + 1
    nc = ncomp(op, dim)
    kr = nb * nc
    c = cells.reshape(-1, nb)
    A = np.zeros((nv * nc, nv * nc))
    for e in range(c.shape[0]):
        m = np.asarray(store[e * kr * kr:(e + 1) * kr * kr], dtype=np.float64).reshape(kr, kr).T
        dof = np.array([c[e, i % nb] * nc + i // nb for i in range(kr)])
        A[np.ix_(dof, dof)] += m
    return A


def to_dense(row_ptr, col_idx, values, n):
    A = np.zeros((n, n), dtype=values.dtype)
    for r in range(n):
        A[r, col_idx[row_ptr[r]:row_ptr[r + 1]]] = values[row_ptr[r]:row_ptr[r + 1]]
    return A


@pytest.mark.parametrize("op", OPS)
@pytest.mark.parametrize("dim,n", [(2, 1), (2, 6), (3, 1), (3, 3)])
def test_plan_pattern_equals_oracle(restatement, op, dim, n):
    v, c = fb.structured_mesh(dim, n, 0.15, 42)
    nv = v.size // dim
    plan = fb.AssemblyPlan(op, dim, c, nv)
    rp, ci = plan.pattern()
    rp2, ci2 = restatement.assembly_pattern(op, dim, c, nv)
    assert plan.rows == nv * ncomp(op, dim)
    assert np.array_equal(rp, rp2) and np.array_equal(ci, ci2)
    # rows sorted, diagonal present
    for r in range(plan.rows):
        row = ci[rp[r]:rp[r + 1]]
        assert np.all(np.diff(row) > 0) and r in row


@pytest.mark.parametrize("dim", [2, 3])
def test_plan_with_unreferenced_vertices_and_shuffled_cells(restatement, dim):
    v, c, _ = fb.mesh_prefix(dim, 37)  # vertex array kept whole: many unreferenced vertices
    nv = v.size // dim
    rng = np.random.default_rng(7)
    cs = c.reshape(-1, dim + 1)[rng.permutation(37)].ravel().copy()
    for cells in (c, cs):
        plan = fb.AssemblyPlan("elasticity", dim, cells, nv)
        rp, ci = plan.pattern()
        rp2, ci2 = restatement.assembly_pattern("elasticity", dim, cells, nv)
        assert np.array_equal(rp, rp2) and np.array_equal(ci, ci2)
    assert np.any(np.diff(rp) == 0)  # empty rows of unreferenced vertices


def test_plan_empty_mesh():
    plan = fb.AssemblyPlan("laplacian", 2, np.zeros(0, dtype=np.int32), 4)
    rp, ci = plan.pattern()
    assert plan.nnz == 0 and np.array_equal(rp, np.zeros(5, dtype=np.int64)) and ci.size == 0


def test_plan_rejects_bad_connectivity():
    v, c = fb.structured_mesh(2, 3)
    nv = v.size // 2
    bad = c.copy()
    bad[3 * 5 + 1] = nv  # cell 5
    with pytest.raises(_lib.InvalidArgument, match="out of range in cell 5") as ei:
        fb.AssemblyPlan("laplacian", 2, bad, nv)
    assert ei.value.cell == 5
    rep = c.copy()
    rep[3 * 2 + 2] = rep[3 * 2]  # cell 2 repeats a vertex
    with pytest.raises(_lib.InvalidArgument, match="repeated vertex in cell 2"):
        fb.AssemblyPlan("laplacian", 2, rep, nv)
    with pytest.raises(_lib.InvalidArgument):
        fb.AssemblyPlan("laplacian", 4, c, nv)


@pytest.mark.parametrize("op", OPS)
@pytest.mark.parametrize("dim,n", [(2, 4), (3, 2)])
@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_oracle_assembly_pinned(restatement, op, dim, n, prec):
    v, c = fb.structured_mesh(dim, n, 0.15, 42)
    nv = v.size // dim
    w = None
    if op == "weighted-laplacian":
        w = 1.0 + v.reshape(-1, dim)[c.reshape(-1, dim + 1), 0].ravel()
    store = restatement.integrate_mesh(op, v, c, dim, bs=1, precision=prec, coeffs=w)
    rp, ci = restatement.assembly_pattern(op, dim, c, nv)
    vals = restatement.assemble(op, dim, c, nv, prec, store, rp, ci)
    n_dof = nv * ncomp(op, dim)
    A = to_dense(rp, ci, vals, n_dof)
    ref = coo_sum(op, dim, c, nv, store)
    tol = 1e-13 if prec == "f64" else 2e-6
    assert np.max(np.abs(A - ref)) <= tol * np.max(np.abs(ref))
    assert np.array_equal(A, A.T)  # bitwise: symmetric element matrices, same summation order
    if op == "laplacian":
        assert np.max(np.abs(A.astype(np.float64).sum(axis=1))) <= 50 * tol * np.max(np.abs(ref))
    if op == "elasticity":
        for comp in range(dim):
            t = np.zeros(n_dof)
            t[comp::dim] = 1.0
            assert np.max(np.abs(A.astype(np.float64) @ t)) <= 50 * tol * np.max(np.abs(ref))
