"""Global CSR assembly on the GPU: the gather kernel's
values are BITWISE the oracle's serial element-order sum over the same store
(every op x dim x precision, host and device buffers, the async API), and at
a BASELINE size the assembled operator keeps the size-independent properties
(bitwise symmetry, zero Laplacian row sums, translation null space)."""
import ctypes as C

import numpy as np
import pytest

import paper_1103_0066_b200 as fb
from paper_1103_0066_b200 import _lib

pytestmark = pytest.mark.gpu
OPS = ["laplacian", "elasticity", "weighted-laplacian"]


def coeffs_for(op, v, c, dim):
    if op != "weighted-laplacian":
        return None
    return np.ascontiguousarray(1.0 + v.reshape(-1, dim)[c.reshape(-1, dim + 1), 0].ravel())


@pytest.mark.parametrize("op", OPS)
@pytest.mark.parametrize("dim,n", [(2, 9), (3, 4)])
@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_assembly_bitwise_vs_oracle(restatement, op, dim, n, prec):
    import torch

    v, c = fb.structured_mesh(dim, n, 0.15, 42)
    nv = v.size // dim
    w = coeffs_for(op, v, c, dim)
    var = fb.make_variant(op, dim, prec, "strict", element_batch_size=16)
    store = fb.integrate_mesh(var, v, c, w)  # host in, host out (padded store)
    want_store = restatement.integrate_mesh(op, v, c, dim, bs=16, precision=prec, coeffs=w)
    assert store.tobytes() == want_store.tobytes()
    plan = fb.AssemblyPlan(op, dim, c, nv)
    rp, ci = plan.pattern()
    want = restatement.assemble(op, dim, c, nv, prec, want_store, rp, ci)
    assert var.path in (0, 3)  # symmetric kernel path: element matrices bitwise symmetric
    for sym in (False, True):
        for diag in (False, True):  # block-diagonal promise (elasticity; a no-op otherwise)
            got_host = plan.assemble(var, store, symmetric=sym, block_diagonal=diag)
            assert got_host.tobytes() == want.tobytes()
            dstore = torch.from_numpy(store).cuda()
            got_dev = plan.assemble(var, dstore, symmetric=sym, block_diagonal=diag)
            assert got_dev.is_cuda and got_dev.cpu().numpy().tobytes() == want.tobytes()
            vals = torch.full((plan.nnz,), float("nan"), dtype=dstore.dtype, device="cuda")
            plan.assemble_async(var, dstore, vals, torch.cuda.current_stream().cuda_stream, symmetric=sym,
                                block_diagonal=diag)
            torch.cuda.synchronize()
            assert vals.cpu().numpy().tobytes() == want.tobytes()


@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_assembly_nonsymmetric_element_matrices(restatement, prec):
    # a non-symmetric K (reference layout, P1 pattern kept): rows != columns
    dim = 3
    k = restatement.build_k("laplacian", dim).copy()
    k[(1 + 2 * 4) * 9 + 0 * 3 + 1] *= 1.5  # block (i=1, j=2), (mu=0, nu=1)
    v, c = fb.structured_mesh(dim, 3, 0.15, 42)
    nv = v.size // dim
    var = fb.make_variant("laplacian", dim, prec, "strict", element_batch_size=8, k=k)
    assert var.path == 1
    store = fb.integrate_mesh(var, v, c)
    plan = fb.AssemblyPlan("laplacian", dim, c, nv)
    rp, ci = plan.pattern()
    want = restatement.assemble("laplacian", dim, c, nv, prec, store, rp, ci)
    assert plan.assemble(var, store).tobytes() == want.tobytes()


def test_assembly_shuffled_cells_and_unreferenced_vertices(restatement):
    v, c, _ = fb.mesh_prefix(3, 1000, 0.1)
    nv = v.size // 3
    cs = c.reshape(-1, 4)[np.random.default_rng(3).permutation(1000)].ravel().copy()
    for cells in (c, cs):
        var = fb.make_variant("elasticity", 3, "f32", "strict", element_batch_size=128)
        store = fb.integrate_mesh(var, v, cells)
        plan = fb.AssemblyPlan("elasticity", 3, cells, nv)
        rp, ci = plan.pattern()
        want = restatement.assemble("elasticity", 3, cells, nv, "f32", store, rp, ci)
        assert plan.assemble(var, store, symmetric=True).tobytes() == want.tobytes()


@pytest.mark.parametrize("op,dim,n", [("laplacian", 2, 7), ("elasticity", 3, 4), ("weighted-laplacian", 3, 3)])
def test_gpu_built_plan_equals_host_plan(op, dim, n):
    import torch

    v, c = fb.structured_mesh(dim, n, 0.15, 42)
    nv = v.size // dim
    cs = c.reshape(-1, dim + 1)[np.random.default_rng(5).permutation(c.size // (dim + 1))].ravel().copy()
    for cells in (c, cs):
        host = fb.AssemblyPlan(op, dim, cells, nv)
        dev = fb.AssemblyPlan(op, dim, torch.from_numpy(cells).cuda(), nv)
        assert dev.rows == host.rows and dev.nnz == host.nnz
        for a, b in zip(dev.pattern(), host.pattern()):
            assert np.array_equal(a, b)
        var = fb.make_variant(op, dim, "f64", "strict", element_batch_size=32)
        w = None
        if op == "weighted-laplacian":
            w = np.ascontiguousarray(1.0 + v.reshape(-1, dim)[cells.reshape(-1, dim + 1), 0].ravel())
        store = torch.from_numpy(fb.integrate_mesh(var, v, cells, w)).cuda()
        assert torch.equal(dev.assemble(var, store), host.assemble(var, store))


def test_gpu_built_plan_rejects_bad_connectivity():
    import torch

    v, c = fb.structured_mesh(3, 2)
    nv = v.size // 3
    bad = c.copy()
    bad[4 * 7 + 2] = -1
    bad[4 * 9 + 0] = nv + 5
    with pytest.raises(_lib.InvalidArgument, match="out of range in cell 7") as ei:
        fb.AssemblyPlan("laplacian", 3, torch.from_numpy(bad).cuda(), nv)
    assert ei.value.cell == 7
    rep = c.copy()
    rep[4 * 3 + 1] = rep[4 * 3 + 3]
    with pytest.raises(_lib.InvalidArgument, match="repeated vertex in cell 3"):
        fb.AssemblyPlan("elasticity", 3, torch.from_numpy(rep).cuda(), nv)


@pytest.mark.parametrize("ids,kind", [((5, 5, -7, 9), "repeated vertex"),     # slot 1 repeats before slot 2 is bad
                                      ((5, -7, 5, 9), "out of range"),        # slot 1 bad before slot 2 repeats
                                      ((11, 4, 11, 10 ** 6), "repeated vertex")])
def test_gpu_and_host_builders_report_the_same_error(ids, kind, monkeypatch):
    """Both plan builders report the lowest bad cell with the failure the host
    builder meets first in slot order, whatever mixes in the cell."""
    import torch

    v, c = fb.structured_mesh(3, 2)
    nv = v.size // 3
    bad = c.copy()
    bad[4 * 6:4 * 7] = ids
    bad[4 * 9 + 1] = nv + 3  # a later bad cell must not win
    msgs = []
    for cells in (bad, torch.from_numpy(bad).cuda()):
        with pytest.raises(_lib.InvalidArgument) as ei:
            fb.AssemblyPlan("laplacian", 3, cells, nv)
        assert ei.value.cell == 6 and kind in str(ei.value)
        msgs.append(str(ei.value))
    assert msgs[0] == msgs[1]


def _raise(plan, var, store):  # fb_assemble with an unknown flag bit
    err = _lib.fb_error()
    rc = plan._lib.fb_assemble(plan._h, var.handle, store.ctypes.data, store.size,
                               np.empty(plan.nnz).ctypes.data, plan.nnz, 6, 0, C.byref(err))
    _lib.raise_for(rc, err)


def test_assembly_validation():
    import torch

    v, c = fb.structured_mesh(2, 4)
    nv = v.size // 2
    plan = fb.AssemblyPlan("laplacian", 2, c, nv)
    var = fb.make_variant("laplacian", 2, "f64", element_batch_size=1)
    store = fb.integrate_mesh(var, v, c)
    with pytest.raises(_lib.InvalidArgument, match="nnz"):
        plan.assemble(var, store, np.empty(plan.nnz + 1))
    with pytest.raises(_lib.InvalidArgument, match="shorter"):
        plan.assemble(var, store[:-1])
    with pytest.raises(_lib.InvalidArgument, match="operator shape"):
        plan.assemble(fb.make_variant("elasticity", 2, "f64", element_batch_size=1),
                      np.zeros(c.size // 3 * 36))
    with pytest.raises(_lib.InvalidArgument, match="flags"):
        _raise(plan, var, store)
    with pytest.raises(_lib.InvalidArgument, match="dimension"):
        plan.assemble(fb.make_variant("laplacian", 3, "f64", element_batch_size=1), np.zeros(10 ** 4))
    del torch


@pytest.mark.parametrize("op,dim,ne,prec", [("laplacian", 3, 1 << 22, "f32"), ("elasticity", 2, 1 << 20, "f32"),
                                            ("elasticity", 3, 1 << 19, "f64")])
def test_assembly_properties_at_size(op, dim, ne, prec):
    import torch

    v, c, _ = fb.mesh_prefix(dim, ne, 0.15 if ne <= (1 << 22) else 0.0)
    nv = v.size // dim
    dv, dc = torch.from_numpy(v).cuda(), torch.from_numpy(c).cuda()
    var = fb.make_variant(op, dim, prec, "strict")
    store = fb.integrate_mesh(var, dv, dc)
    plan = fb.AssemblyPlan(op, dim, c, nv)
    vals = plan.assemble(var, store, symmetric=True)
    rp, ci = plan.pattern()
    rows = torch.repeat_interleave(torch.arange(plan.rows, device="cuda"), torch.from_numpy(np.diff(rp)).cuda())
    cols = torch.from_numpy(ci).cuda().long()
    # bitwise symmetry: A[r, c] == A[c, r] for every stored entry
    key = rows * plan.rows + cols
    tkey = cols * plan.rows + rows
    order = torch.argsort(key)
    pos = torch.searchsorted(key[order], tkey)
    assert torch.equal(key[order][pos], tkey)
    assert torch.equal(vals[order][pos], vals)
    scale = vals.abs().max().item()
    nc = dim if op == "elasticity" else 1
    v64 = vals.double()
    for comp in range(nc):
        t = (cols % nc == comp).double()  # translation in component `comp`
        r = torch.zeros(plan.rows, dtype=torch.float64, device="cuda").index_add_(0, rows, v64 * t)
        assert r.abs().max().item() <= (1e-4 if prec == "f32" else 1e-12) * scale


def fan_mesh(dim, m):
    """m elements around a hub (2D) or an axis (3D): hub vertices of degree
    m + dim - 1, above every kernel's shared-memory slot count."""
    t = 2 * np.pi * np.arange(m) / m
    if dim == 2:
        v = np.concatenate([[0.0, 0.0], np.stack([np.cos(t), np.sin(t)], 1).ravel()])
        c = np.array([[0, 1 + i, 1 + (i + 1) % m] for i in range(m)], dtype=np.int32)
    else:
        ring = np.stack([np.cos(t), np.sin(t), 0.3 + 0.1 * np.sin(3 * t)], 1)
        v = np.concatenate([[0.0, 0.0, 0.0, 0.0, 0.0, 1.0], ring.ravel()])
        c = np.array([[0, 1, 2 + i, 2 + (i + 1) % m] for i in range(m)], dtype=np.int32)
    x = v.reshape(-1, dim)[c]
    j = (x[:, 1:] - x[:, :1]).transpose(0, 2, 1)
    neg = np.linalg.det(j) < 0
    c[neg, -2], c[neg, -1] = c[neg, -1].copy(), c[neg, -2].copy()
    return np.ascontiguousarray(v), np.ascontiguousarray(c.ravel())


def _packed_case(var, op, dim, v, c, prec, bs, offset=0):
    """(want, got): assemble(integrate_batches(G)) vs assemble_packed(G);
    offset > 0 places G that many scalars into a buffer (misaligned)."""
    import torch

    nv, ne = v.size // dim, c.size // (dim + 1)
    w = coeffs_for(op, v, c, dim)
    dv, dc = torch.from_numpy(v).cuda(), torch.from_numpy(c).cuda()
    dw = torch.from_numpy(w).cuda() if w is not None else None
    g = fb.pack_geometry(dv, dc, dim, bs, prec)
    if offset:
        buf = torch.empty(g.numel() + offset, dtype=g.dtype, device="cuda")
        buf[offset:] = g
        g = buf[offset:]
    store = fb.integrate_batches(var, g, ne, dw)
    plan = fb.AssemblyPlan(op, dim, dc, nv)
    want = plan.assemble(var, store)
    got = torch.full_like(want, float("nan"))
    plan.assemble_packed_async(var, g, got, dw, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    # synchronous API: host buffers (staged) and device tensors
    host = plan.assemble_packed(var, g.cpu().numpy(), w)
    assert host.tobytes() == want.cpu().numpy().tobytes()
    assert torch.equal(plan.assemble_packed(var, g, dw), want)
    # mixed residency: host G and coefficients, device values
    mixed = torch.full_like(want, float("nan"))
    plan.assemble_packed(var, g.cpu().numpy(), w, values=mixed)
    assert torch.equal(mixed, want)
    return want, got


@pytest.mark.parametrize("op", OPS)
@pytest.mark.parametrize("dim,n", [(2, 9), (3, 4)])
@pytest.mark.parametrize("prec", ["f32", "f64"])
@pytest.mark.parametrize("mode", ["strict", "fast"])
def test_packed_assembly_bitwise(op, dim, n, prec, mode):
    # assembly straight from packed G == assembly of the integrate_batches store
    v, c = fb.structured_mesh(dim, n, 0.15, 42)
    var = fb.make_variant(op, dim, prec, mode, element_batch_size=16)
    want, got = _packed_case(var, op, dim, v, c, prec, 16)
    assert got.cpu().numpy().tobytes() == want.cpu().numpy().tobytes()
    # G not 16-byte aligned (scalar reads) and G of unpadded length (the
    # last element's covering words would pass the end: read scalar-wise)
    want, got = _packed_case(var, op, dim, v, c, prec, 16, offset=1)
    assert got.cpu().numpy().tobytes() == want.cpu().numpy().tobytes()
    var1 = fb.make_variant(op, dim, prec, mode, element_batch_size=1)
    want, got = _packed_case(var1, op, dim, v, c, prec, 1)
    assert got.cpu().numpy().tobytes() == want.cpu().numpy().tobytes()


@pytest.mark.parametrize("op", OPS)
@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_packed_assembly_high_degree_and_general_k(restatement, op, dim, prec):
    import torch

    # hub vertices beyond the shared-memory slots accumulate in global memory
    v, c = fan_mesh(dim, 40)
    var = fb.make_variant(op, dim, prec, "strict", element_batch_size=8)
    want, got = _packed_case(var, op, dim, v, c, prec, 8)
    assert got.cpu().numpy().tobytes() == want.cpu().numpy().tobytes()
    # a non-symmetric K with the P1 pattern (path 1)
    k = restatement.build_k(op, dim).copy()
    nb = dim + 1
    nc = dim if op == "elasticity" else 1
    kr = nb * nc
    k4 = k.reshape(kr, kr, -1, dim * dim)  # [j][i][coefficient][mu*dim + nu]
    for comp in range(nc):  # (a=1, b=2, mu=0, nu=1) in every component block
        k4[2 + comp * nb, 1 + comp * nb, 0, 1] *= 1.5
    var = fb.make_variant(op, dim, prec, "strict", element_batch_size=8, k=k)
    assert var.path == 1
    v, c = fb.structured_mesh(dim, 3, 0.15, 7)
    want, got = _packed_case(var, op, dim, v, c, prec, 8)
    assert got.cpu().numpy().tobytes() == want.cpu().numpy().tobytes()
    del torch


@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_block_diagonal_store_assembly_hub_vertices(restatement, dim, prec):
    """Block-diagonal reads with hub vertices beyond the shared-memory slots
    (accumulated in the output rows, then expanded over the components)."""
    v, c = fan_mesh(dim, 40)
    nv = v.size // dim
    var = fb.make_variant("elasticity", dim, prec, "strict", element_batch_size=8)
    store = fb.integrate_mesh(var, v, c)
    plan = fb.AssemblyPlan("elasticity", dim, c, nv)
    rp, ci = plan.pattern()
    want = restatement.assemble("elasticity", dim, c, nv, prec, store, rp, ci)
    for sym in (False, True):
        assert plan.assemble(var, store, symmetric=sym, block_diagonal=True).tobytes() == want.tobytes()


def test_packed_assembly_validation(restatement):
    import torch

    v, c = fb.structured_mesh(3, 2)
    nv, ne = v.size // 3, c.size // 4
    plan = fb.AssemblyPlan("laplacian", 3, c, nv)
    var = fb.make_variant("laplacian", 3, "f64", element_batch_size=1)
    vals = torch.empty(plan.nnz, dtype=torch.float64, device="cuda")
    g = torch.zeros(ne * 9, dtype=torch.float64, device="cuda")
    with pytest.raises(_lib.InvalidArgument, match="packed geometry shorter"):
        plan.assemble_packed_async(var, g[:-1], vals)
    wvar = fb.make_variant("weighted-laplacian", 3, "f64", element_batch_size=1)
    with pytest.raises(_lib.InvalidArgument, match="nodal coefficients"):
        plan.assemble_packed_async(wvar, g, vals)
    dense_k = restatement.build_k("laplacian", 3).copy()
    dense_k[dense_k == 0] = 0.25  # breaks the P1 pattern: dense path
    dvar = fb.make_variant("laplacian", 3, "f64", element_batch_size=1, k=dense_k)
    assert dvar.path == 2
    with pytest.raises(_lib.InvalidArgument, match="P1 sparsity"):
        plan.assemble_packed_async(dvar, g, vals)


@pytest.mark.parametrize("op,dim", [("laplacian", 2), ("elasticity", 3), ("weighted-laplacian", 3)])
def test_assembly_of_an_empty_mesh(op, dim):
    import torch

    cells = np.zeros(0, dtype=np.int32)
    for c in (cells, torch.from_numpy(cells).cuda()):
        plan = fb.AssemblyPlan(op, dim, c, 5)
        nc = dim if op == "elasticity" else 1
        assert plan.rows == 5 * nc and plan.nnz == 0
        rp, ci = plan.pattern()
        assert rp.tolist() == [0] * (5 * nc + 1) and ci.size == 0
        var = fb.make_variant(op, dim, "f64", element_batch_size=4)
        assert plan.assemble(var, np.zeros(0)).size == 0
        coeffs = np.zeros(0) if op == "weighted-laplacian" else None
        assert plan.assemble_packed(var, np.zeros(0), coeffs).size == 0
        vals = torch.empty(0, dtype=torch.float64, device="cuda")
        plan.assemble_packed_async(var, torch.empty(0, dtype=torch.float64, device="cuda"), vals,
                                   torch.empty(0, dtype=torch.float64, device="cuda") if coeffs is not None else None,
                                   torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()


@pytest.mark.parametrize("op,dim", [("elasticity", 3), ("laplacian", 2)])
def test_large_host_connectivity_is_planned_on_the_gpu(op, dim, monkeypatch):
    import torch

    # >= 65,536 elements of host connectivity: uploaded and planned on the
    # GPU; the plan equals the host builder's (FB_PLAN_HOST) array for array
    v, c, _ = fb.mesh_prefix(dim, 70000, 0.1)
    cs = c.reshape(-1, dim + 1)[np.random.default_rng(2).permutation(70000)].ravel().copy()
    nv = v.size // dim
    for cells in (c, cs):
        auto = fb.AssemblyPlan(op, dim, cells, nv)
        monkeypatch.setenv("FB_PLAN_HOST", "1")
        host = fb.AssemblyPlan(op, dim, cells, nv)
        monkeypatch.delenv("FB_PLAN_HOST")
        assert auto.nnz == host.nnz
        for x, y in zip(auto.pattern(), host.pattern()):
            assert np.array_equal(x, y)
        var = fb.make_variant(op, dim, "f32", "strict")
        store = fb.integrate_mesh(var, torch.from_numpy(v).cuda(), torch.from_numpy(cells).cuda())
        assert torch.equal(auto.assemble(var, store, symmetric=True), host.assemble(var, store, symmetric=True))
    bad = c.copy()
    bad[(dim + 1) * 60001 + 1] = nv + 3
    with pytest.raises(_lib.InvalidArgument, match="out of range in cell 60001"):
        fb.AssemblyPlan(op, dim, bad, nv)
