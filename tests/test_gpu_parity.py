"""GPU parity: the CUDA path (through the C ABI) against the oracle.

Bar:
* strict mode: BITWISE equal to the reference engine (pack_geometry +
  integrate_batches) -- checked against the C restatement on seeded jittered
  meshes and against golden fixtures produced by the unmodified reference;
* fast mode: normwise per-element error vs the FP64 direct-quadrature oracle
  <= 1e-13 (f64) and <= 5e-6 (f32);
* connectivity / indexing / padding: exact.
"""
import os

import numpy as np
import pytest

import paper_1103_0066_b200 as fb
from oracle.oracle import OPS, krows, normwise_error

pytestmark = pytest.mark.gpu

TOL = {"f64": 1e-13, "f32": 5e-6}
REF_TRI = np.array([[1.0, -0.5, -0.5], [-0.5, 0.5, 0.0], [-0.5, 0.0, 0.5]])


def mesh(dim, n, jitter=0.15, seed=42):
    return fb.structured_mesh(dim, n, jitter, seed)


def coeffs_for(op, v, c, dim):
    if op != "weighted-laplacian":
        return None
    # reference default_coefficient_field: w = 1 + x0 at each cell vertex (bench.cpp:19-30)
    vv = v.reshape(-1, dim)
    return np.ascontiguousarray((1.0 + vv[c.reshape(-1, dim + 1), 0]).ravel())


@pytest.mark.parametrize("name", ["m2", "m3", "m2b"])
@pytest.mark.parametrize("op", list(OPS))
@pytest.mark.parametrize("prec", ["f32", "f64"])
@pytest.mark.parametrize("store", ["auto", "staged", "tma", "direct"])
def test_strict_matches_reference_golden(golden, name, op, prec, store):
    dim = 3 if name == "m3" else 2
    bs = {"m2": 16, "m3": 7, "m2b": 128}[name]
    v, c = golden[f"{name}_vertices"], golden[f"{name}_cells"]
    w = golden[f"{name}_coeffs"] if op == "weighted-laplacian" else None
    var = fb.make_variant(op, dim, prec, "strict", element_batch_size=bs, store=store)
    got = fb.integrate_mesh(var, v, c, w)
    p = 0 if prec == "f32" else 1
    want = golden[f"{name}_store_{op}_p{p}"]
    assert got.dtype == want.dtype and got.size == want.size
    assert got.tobytes() == want.tobytes()


@pytest.mark.parametrize("dim,n", [(2, 60), (3, 13)])
@pytest.mark.parametrize("op", list(OPS))
@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_strict_bitwise_vs_restatement(restatement, dim, n, op, prec):
    v, c = mesh(dim, n, 0.15, 42)
    w = coeffs_for(op, v, c, dim)
    for bs in (128, 100):
        var = fb.make_variant(op, dim, prec, "strict", element_batch_size=bs)
        assert var.path == 3  # P1 structure, symmetry, uniform magnitude validated
        got = fb.integrate_mesh(var, v, c, w)
        want = restatement.integrate_mesh(op, v, c, dim, bs=bs, precision=prec, coeffs=w)
        assert got.tobytes() == want.tobytes()


@pytest.mark.parametrize("dim,n", [(2, 40), (3, 9)])
@pytest.mark.parametrize("op", list(OPS))
@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_fast_within_tolerance_of_direct_oracle(restatement, dim, n, op, prec):
    v, c = mesh(dim, n, 0.15, 42)
    w = coeffs_for(op, v, c, dim)
    var = fb.make_variant(op, dim, prec, "fast", element_batch_size=64)
    got = fb.integrate_mesh(var, v, c, w)
    ne = c.size // (dim + 1)
    kr = krows(op, dim)
    a = got[: ne * kr * kr].reshape(ne, kr, kr).transpose(0, 2, 1)  # store is j-major
    want = restatement.direct_mesh(op, v, c, dim, w)
    assert normwise_error(a, want) <= TOL[prec]
    # strict is also within the same tolerance (sanity of the oracle metric)
    s = fb.integrate_mesh(fb.make_variant(op, dim, prec, "strict", element_batch_size=64), v, c, w)
    assert normwise_error(s[: ne * kr * kr].reshape(ne, kr, kr).transpose(0, 2, 1), want) <= TOL[prec]


def test_reference_triangle_bitwise():
    var = fb.make_variant("laplacian", 2, "f64", element_batch_size=1)
    out = fb.integrate_mesh(var, np.array([0.0, 0, 1, 0, 0, 1]), np.array([0, 1, 2], dtype=np.int32))
    assert np.array_equal(fb.unpack_element_matrix(out, 3, 0), REF_TRI)


def test_synthetic_packed_geometry(golden):
    # test_engine.cpp:337-378 through the G-input path, padded batch, exact
    var = fb.make_variant("laplacian", 2, "f64", element_batch_size=4, num_concurrent_elements=2,
                          interleave_stores=True, loop_unroll=True)
    assert var.description == "bs4_ce2_is_unroll"
    out = fb.integrate_batches(var, golden["synthetic_G"], 5)
    assert out.size == 72
    for e in range(5):
        assert np.array_equal(fb.unpack_element_matrix(out, 3, e), (e + 1) * REF_TRI)
    assert out.tobytes() == golden["synthetic_store"].tobytes()


@pytest.mark.parametrize("dim,n", [(2, 30), (3, 7)])
@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_pack_and_packed_path_bitwise(restatement, dim, n, prec):
    v, c = mesh(dim, n, 0.15, 3)
    bs = 32
    g = fb.pack_geometry(v, c, dim, bs, prec)
    assert g.tobytes() == restatement.pack_geometry(v, c, dim, bs, prec).tobytes()
    ne = c.size // (dim + 1)
    for op in OPS:
        w = coeffs_for(op, v, c, dim)
        var = fb.make_variant(op, dim, prec, element_batch_size=bs)
        got = fb.integrate_batches(var, g, ne, w)
        want = restatement.integrate_packed(op, dim, g, ne, bs, prec, coeffs=w)
        assert got.tobytes() == want.tobytes()
        # fused == pack + integrate, bitwise
        assert fb.integrate_mesh(var, v, c, w).tobytes() == got.tobytes()


@pytest.mark.parametrize("op", list(OPS))
def test_dense_fallback_for_unstructured_k(restatement, op):
    dim = 2
    v, c = mesh(dim, 12, 0.1, 5)
    w = coeffs_for(op, v, c, dim)
    k = fb.build_analytic_tensor(op, dim).copy()
    kr, nc = krows(op, dim), (dim + 1 if op == "weighted-laplacian" else 1)
    k[((1 + 1 * kr) * nc) * dim * dim + 1] = 0.125  # block (1,1), mu=0 nu=1: a structural zero
    for prec in ("f32", "f64"):
        var = fb.make_variant(op, dim, prec, k=k, element_batch_size=16)
        assert var.path == 2
        got = fb.integrate_mesh(var, v, c, w)
        g = restatement.pack_geometry(v, c, dim, 16, prec)
        want = restatement.integrate_packed(op, dim, g, c.size // 3, 16, prec, k=k, coeffs=w)
        assert got.tobytes() == want.tobytes()


@pytest.mark.parametrize("op", list(OPS))
@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_symmetric_nonuniform_k_takes_sparse_sym_path(restatement, op, prec):
    dim = 3
    v, c = mesh(dim, 4, 0.1, 5)
    w = coeffs_for(op, v, c, dim)
    k = fb.build_analytic_tensor(op, dim).copy()
    kr, nc, dd = krows(op, dim), (dim + 1 if op == "weighted-laplacian" else 1), dim * dim
    for comp in range(dim if op == "elasticity" else 1):  # scale block (a=1,b=1) on every component
        i = 1 + comp * (dim + 1)
        k[(i + i * kr) * nc * dd:(i + i * kr + 1) * nc * dd] *= 3.0
    var = fb.make_variant(op, dim, prec, k=k, element_batch_size=8)
    assert var.path == 0
    got = fb.integrate_mesh(var, v, c, w)
    g = restatement.pack_geometry(v, c, dim, 8, prec)
    want = restatement.integrate_packed(op, dim, g, c.size // 4, 8, prec, k=k, coeffs=w)
    assert got.tobytes() == want.tobytes()
    assert fb.integrate_batches(var, g, c.size // 4, w).tobytes() == want.tobytes()


def test_nonsymmetric_k_takes_sparse_path(restatement):
    dim = 3
    v, c = mesh(dim, 4, 0.1, 5)
    k = fb.build_analytic_tensor("laplacian", dim).copy()
    k[(0 + 1 * 4) * 9 + 3] *= 2.0  # block (0,1), mu=1 nu=0: still on the P1 pattern, asymmetric
    var = fb.make_variant("laplacian", dim, "f64", k=k, element_batch_size=8)
    assert var.path == 1
    got = fb.integrate_mesh(var, v, c)
    g = restatement.pack_geometry(v, c, dim, 8, 1)
    want = restatement.integrate_packed("laplacian", dim, g, c.size // 4, 8, 1, k=k)
    assert got.tobytes() == want.tobytes()


@pytest.mark.parametrize("ne", [1, 2, 287, 288, 289, 1000, 4097])
@pytest.mark.parametrize("dim", [2, 3])
def test_ragged_sizes_and_padding(restatement, ne, dim):
    v, c, _ = fb.mesh_prefix(dim, ne, 0.1, 11)
    for prec, op in (("f32", "laplacian"), ("f64", "elasticity"), ("f32", "elasticity"), ("f64", "laplacian")):
        for bs in (1, 7, 128):
            var = fb.make_variant(op, dim, prec, element_batch_size=bs)
            got = fb.integrate_mesh(var, v, c)
            want = restatement.integrate_mesh(op, v, c, dim, bs=bs, precision=prec)
            assert got.tobytes() == want.tobytes()  # padding slots replicate the last element


def test_empty_mesh():
    var = fb.make_variant("laplacian", 3, "f32")
    out = fb.integrate_mesh(var, np.zeros(12), np.zeros(0, dtype=np.int32))
    assert out.size == 0
    wv = fb.make_variant("weighted-laplacian", 2, "f64")
    with pytest.raises(ValueError, match="zero elements"):
        fb.integrate_mesh(wv, np.zeros(6), np.zeros(0, dtype=np.int32), np.zeros(3))


def test_degenerate_cell_reports_lowest_index():
    v, c = mesh(2, 8, 0.0)
    c = c.copy()
    c[5 * 3:5 * 3 + 3] = c[5 * 3:5 * 3 + 3][[0, 2, 1]]  # invert cell 5
    c[40 * 3:40 * 3 + 3] = c[40 * 3:40 * 3 + 3][[0, 2, 1]]
    for mode in ("strict", "fast"):
        var = fb.make_variant("laplacian", 2, "f64", mode)
        with pytest.raises(RuntimeError, match=r"degenerate element: det\(J\) <= 0 in cell 5") as ei:
            fb.integrate_mesh(var, v, c)
        assert ei.value.cell == 5


def test_out_of_range_vertex_is_reported():
    v, c = mesh(3, 2, 0.0)
    c = c.copy()
    c[9] = 10_000
    var = fb.make_variant("laplacian", 3, "f64")
    with pytest.raises(ValueError, match="out of range in cell 2"):
        fb.integrate_mesh(var, v, c)


def test_argument_validation_precedes_compute():
    v, c = mesh(2, 3)
    lap = fb.make_variant("laplacian", 2, "f64")
    with pytest.raises(ValueError, match="form takes no coefficient field"):
        fb.integrate_mesh(lap, v, c, np.ones(c.size))
    wl = fb.make_variant("weighted-laplacian", 2, "f64")
    with pytest.raises(ValueError, match="form requires a coefficient field"):
        fb.integrate_mesh(wl, v, c)
    import ctypes as C

    from paper_1103_0066_b200 import _lib

    l3 = fb.make_variant("laplacian", 3, "f64")
    mv = fb.engine.mesh_view(v, c, 2)  # a 2D mesh handed to a 3D variant
    out = np.zeros(l3.store_length(c.size // 3))
    err = _lib.fb_error()
    rc = _lib.load().fb_integrate_mesh(l3.handle, C.byref(mv), None, out.ctypes.data, out.size, None, 0,
                                       C.byref(err))
    assert rc == _lib.FB_ERR_INVALID_ARGUMENT
    assert err.message.decode() == "geometry dimension does not match form"


def test_device_tensors_and_async_api(restatement):
    import torch

    dim, op, prec = 3, "elasticity", "f32"
    v, c = mesh(dim, 6, 0.15, 1)
    var = fb.make_variant(op, dim, prec)
    dv, dc = torch.from_numpy(v).cuda(), torch.from_numpy(c).cuda()
    out = fb.integrate_mesh(var, dv, dc)
    assert out.is_cuda
    want = restatement.integrate_mesh(op, v, c, dim, bs=128, precision=prec)
    assert out.cpu().numpy().tobytes() == want.tobytes()
    out2 = torch.empty_like(out)
    status = torch.empty(2, dtype=torch.int64, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    fb.status_reset(status, s)
    fb.integrate_mesh_async(var, dv, dc, out2, status, s)
    fb.status_check(status, s)
    assert torch.equal(out, out2)


def test_multi_device_sharding_concatenates():
    """devices=[0,0,0]: three contiguous tile-aligned shards on one GPU must
    concatenate to the single-launch store bitwise."""
    dim = 2
    v, c, _ = fb.mesh_prefix(dim, 100_003, 0.1, 2)
    for op, prec in (("elasticity", "f32"), ("laplacian", "f64")):
        var = fb.make_variant(op, dim, prec, element_batch_size=64)
        one = fb.integrate_mesh(var, v, c)
        three = fb.integrate_mesh(var, v, c, devices=[0, 0, 0])
        assert one.tobytes() == three.tobytes()


def test_variant_invariance_bitwise():
    # acceptance.cpp:175-215: every tuning axis is value-neutral
    v, c = mesh(2, 10, 0.15, 42)
    base = fb.integrate_mesh(fb.make_variant("laplacian", 2, "f32", element_batch_size=16), v, c)
    ne = c.size // 3
    for bs in (16, 32):
        for ce in (1, 2, 4):
            for is_ in (False, True):
                for ur in (False, True):
                    for store in ("auto", "staged", "tma", "direct"):
                        var = fb.make_variant("laplacian", 2, "f32", element_batch_size=bs,
                                              num_concurrent_elements=ce, interleave_stores=is_,
                                              loop_unroll=ur, store=store)
                        got = fb.integrate_mesh(var, v, c)
                        assert got[: ne * 9].tobytes() == base[: ne * 9].tobytes()


@pytest.mark.parametrize("dim,n", [(2, 30), (3, 9)])
@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_pack_geometry_async_bitwise(restatement, dim, n, prec):
    import torch

    v, c = mesh(dim, n)
    ne = c.size // (dim + 1)
    want = restatement.pack_geometry(v, c, dim, 32, prec)
    g = torch.empty(want.size, dtype=torch.float32 if prec == "f32" else torch.float64, device="cuda")
    st = torch.empty(2, dtype=torch.int64, device="cuda")
    sid = torch.cuda.current_stream().cuda_stream
    fb.status_reset(st, sid)
    fb.pack_geometry_async(torch.from_numpy(v).cuda(), torch.from_numpy(c).cuda(), dim, g, st, 32, prec, sid)
    fb.status_check(st, sid)
    assert g.cpu().numpy().tobytes() == want.tobytes()
    assert ne > 0


@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_unaligned_device_outputs(restatement, prec):
    """Caller buffers that are scalar- but not 16-byte-aligned take the
    per-lane store path (scalar stores) and give the same bits."""
    import torch

    dt = torch.float32 if prec == "f32" else torch.float64
    st = torch.empty(2, dtype=torch.int64, device="cuda")
    sid = torch.cuda.current_stream().cuda_stream
    for op, dim, n in (("laplacian", 3, 6), ("elasticity", 2, 12)):
        v, c = mesh(dim, n)
        dv, dc = torch.from_numpy(v).cuda(), torch.from_numpy(c).cuda()
        var = fb.make_variant(op, dim, prec, "strict", element_batch_size=8)
        ne = c.size // (dim + 1)
        want = restatement.integrate_mesh(op, v, c, dim, bs=8, precision=prec)
        buf = torch.empty(var.store_length(ne) + 1, dtype=dt, device="cuda")
        out = buf[1:]
        fb.status_reset(st, sid)
        fb.integrate_mesh_async(var, dv, dc, out, st, sid)
        fb.status_check(st, sid)
        assert out.cpu().numpy().tobytes() == want.tobytes()
        gwant = restatement.pack_geometry(v, c, dim, 8, prec)
        gbuf = torch.empty(gwant.size + 1, dtype=dt, device="cuda")
        fb.pack_geometry_async(dv, dc, dim, gbuf[1:], st, 8, prec, sid)
        fb.status_check(st, sid)
        assert gbuf[1:].cpu().numpy().tobytes() == gwant.tobytes()


@pytest.mark.parametrize("op,mode", [("laplacian", "strict"), ("laplacian", "fast"), ("weighted-laplacian", "strict")])
def test_3d_fp32_direct_stores_and_their_alignment_fallbacks(restatement, op, mode):
    """3D Laplacian-shaped FP32 stores leave by per-lane 32-byte stores when
    the output is 32-byte aligned; 16- but not 32-byte aligned outputs take
    the staged copy, 4-byte aligned ones scalar stores -- every offset gives
    the same bits (strict: the reference's; fast: the aligned run's)."""
    import torch

    v, c = mesh(3, 6)
    ne = c.size // 4
    w = None
    if op == "weighted-laplacian":
        w = np.ascontiguousarray(1.0 + v.reshape(-1, 3)[c.reshape(-1, 4), 0].ravel())
    var = fb.make_variant(op, 3, "f32", mode, element_batch_size=32)
    dv, dc = torch.from_numpy(v).cuda(), torch.from_numpy(c).cuda()
    dw = None if w is None else torch.from_numpy(w).cuda()
    st = torch.empty(2, dtype=torch.int64, device="cuda")
    sid = torch.cuda.current_stream().cuda_stream
    n = var.store_length(ne)
    buf = torch.empty(n + 8, dtype=torch.float32, device="cuda")
    assert buf.data_ptr() % 32 == 0
    got = []
    for off in (0, 4, 1):  # 32-byte, 16-byte, 4-byte aligned
        out = buf[off:off + n]
        out.fill_(float("nan"))
        fb.status_reset(st, sid)
        fb.integrate_mesh_async(var, dv, dc, out, st, sid, coefficients=dw)
        fb.status_check(st, sid)
        got.append(out.cpu().numpy().tobytes())
    assert got[0] == got[1] == got[2]
    if mode == "strict":
        assert got[0] == restatement.integrate_mesh(op, v, c, 3, bs=32, precision="f32", coeffs=w).tobytes()


def test_multi_device_with_device_resident_buffers(restatement):
    """Shards over a device list with device-resident inputs and output: each
    shard stages its slice from / to wherever the buffers live (peer copies
    across GPUs; here all on GPU 0) and the store concatenates bitwise."""
    import torch

    v, c = mesh(3, 7)
    want = restatement.integrate_mesh("elasticity", v, c, 3, bs=128, precision="f32")
    var = fb.make_variant("elasticity", 3, "f32", "strict", element_batch_size=128)
    out = torch.empty(want.size, dtype=torch.float32, device="cuda")
    fb.integrate_mesh(var, torch.from_numpy(v).cuda(), torch.from_numpy(c).cuda(), out=out, devices=[0, 0, 0])
    assert out.cpu().numpy().tobytes() == want.tobytes()
    hout = np.empty(want.size, dtype=np.float32)
    fb.integrate_mesh(var, torch.from_numpy(v).cuda(), c, out=hout, devices=[0, 0])
    assert hout.tobytes() == want.tobytes()


@pytest.mark.parametrize("dim,n", [(2, 9), (3, 4)])
def test_unaligned_inputs_take_the_scalar_load_paths(restatement, dim, n):
    """Vertex / connectivity arrays that are not 16-byte aligned (2D: no
    double2 vertex loads; 3D: no int4 connectivity loads) give the same bits."""
    import torch

    v, c = mesh(dim, n)
    ne = c.size // (dim + 1)
    vb = torch.empty(v.size + 1, dtype=torch.float64, device="cuda")
    cb = torch.empty(c.size + 1, dtype=torch.int32, device="cuda")
    vb[1:] = torch.from_numpy(v)
    cb[1:] = torch.from_numpy(c)
    st = torch.empty(2, dtype=torch.int64, device="cuda")
    sid = torch.cuda.current_stream().cuda_stream
    for op, prec in (("laplacian", "f64"), ("elasticity", "f32")):
        var = fb.make_variant(op, dim, prec, "strict", element_batch_size=16)
        want = restatement.integrate_mesh(op, v, c, dim, bs=16, precision=prec)
        out = torch.empty(want.size, dtype=torch.float32 if prec == "f32" else torch.float64, device="cuda")
        fb.status_reset(st, sid)
        fb.integrate_mesh_async(var, vb[1:], cb[1:], out, st, sid)
        fb.status_check(st, sid)
        assert out.cpu().numpy().tobytes() == want.tobytes()
        gw = restatement.pack_geometry(v, c, dim, 16, prec)
        g = torch.empty(gw.size, dtype=out.dtype, device="cuda")
        fb.pack_geometry_async(vb[1:], cb[1:], dim, g, st, 16, prec, sid)
        fb.status_check(st, sid)
        assert g.cpu().numpy().tobytes() == gw.tobytes()
    assert ne > 0


def test_async_api_is_cuda_graph_capturable(restatement):
    """The device-resident entry points enqueue kernels only (no allocation,
    no synchronisation), so a whole mesh -> matrices -> CSR pipeline can be
    captured once in a CUDA graph and replayed."""
    import torch

    v, c = mesh(3, 5)
    nv, ne = v.size // 3, c.size // 4
    var = fb.make_variant("laplacian", 3, "f32", "strict", element_batch_size=128)
    dv, dc = torch.from_numpy(v).cuda(), torch.from_numpy(c).cuda()
    out = torch.empty(var.store_length(ne), dtype=torch.float32, device="cuda")
    st = torch.empty(2, dtype=torch.int64, device="cuda")
    plan = fb.AssemblyPlan("laplacian", 3, dc, nv)
    vals = torch.empty(plan.nnz, dtype=torch.float32, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):  # warm-up: first-call host setup (occupancy cache)
        fb.status_reset(st, s.cuda_stream)
        fb.integrate_mesh_async(var, dv, dc, out, st, s.cuda_stream)
        plan.assemble_async(var, out, vals, s.cuda_stream, symmetric=True)
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    out.zero_()
    vals.zero_()
    with torch.cuda.graph(g, stream=s):
        fb.integrate_mesh_async(var, dv, dc, out, st, s.cuda_stream)
        plan.assemble_async(var, out, vals, s.cuda_stream, symmetric=True)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    want = restatement.integrate_mesh("laplacian", v, c, 3, bs=128, precision="f32")
    assert out.cpu().numpy().tobytes() == want.tobytes()
    rp, ci = plan.pattern()
    assert vals.cpu().numpy().tobytes() == restatement.assemble("laplacian", 3, c, nv, "f32", want, rp, ci).tobytes()


def test_library_allocated_device_store(restatement):
    """fb_device_alloc / fb_free: a library-allocated device store used as the
    output of the async entry point (read back with the CUDA runtime)."""
    import ctypes
    import glob

    import nvidia.cuda_runtime
    import torch

    cudart = ctypes.CDLL(glob.glob(os.path.join(list(nvidia.cuda_runtime.__path__)[0], "lib", "libcudart.so*"))[0])
    lib = fb.engine.L.load()
    v, c = mesh(2, 6)
    ne = c.size // 3
    var = fb.make_variant("elasticity", 2, "f64", "strict", element_batch_size=8)
    n = var.store_length(ne)
    err = fb.engine.L.fb_error()
    p = lib.fb_device_alloc(n * 8, 0, ctypes.byref(err))
    assert p and p % 256 == 0
    st = torch.empty(2, dtype=torch.int64, device="cuda")
    dv, dc = torch.from_numpy(v).cuda(), torch.from_numpy(c).cuda()
    mv = fb.engine.mesh_view(dv, dc, 2)
    sid = torch.cuda.current_stream().cuda_stream
    fb.status_reset(st, sid)
    rc = lib.fb_integrate_mesh_async(var.handle, ctypes.byref(mv), None, ctypes.c_void_p(p), n, st.data_ptr(),
                                     ctypes.c_void_p(sid), ctypes.byref(err))
    assert rc == 0, err.message
    fb.status_check(st, sid)
    host = np.empty(n, dtype=np.float64)
    assert cudart.cudaMemcpy(ctypes.c_void_p(host.ctypes.data), ctypes.c_void_p(p), ctypes.c_size_t(n * 8), 2) == 0
    want = restatement.integrate_mesh("elasticity", v, c, 2, bs=8, precision="f64")
    assert host.tobytes() == want.tobytes()
    assert lib.fb_free(ctypes.c_void_p(p), ctypes.byref(err)) == 0


def test_launch_counter_counts_kernels():
    v, c = mesh(2, 4)
    var = fb.make_variant("laplacian", 2, "f64")
    n0 = fb.launch_counter()
    fb.integrate_mesh(var, v, c)
    assert fb.launch_counter() - n0 == 1
