"""The C-ABI boundary on CPU: the library loads, exports every symbol the
header declares, its pure host functions reproduce the reference's goldens,
specialization validates like the reference (same exception texts), and the
integration entry points fail loudly -- never fall back -- without a GPU."""
import os
import re

import numpy as np
import pytest

import paper_1103_0066_b200 as fb
from paper_1103_0066_b200 import _lib
from oracle.oracle import OPS

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "fembatch_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(fb_[a-z0-9_]+)\s*\(", text)))


def test_every_declared_symbol_is_exported_and_bound():
    lib = _lib.load()
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(_lib.SIGNATURES) == syms  # the Python binding covers the whole ABI
    assert lib.fb_abi_version() == 1


def test_flop_and_index_goldens():
    # reference tests/test_engine.cpp:309-318 and :46-57
    assert fb.flop_count("laplacian", 3, 1) == 288
    assert fb.flop_count("elasticity", 2, 1) == 288
    assert fb.flop_count("weighted-laplacian", 2, 1) == 270
    assert fb.flop_count("laplacian", 3, 0) == 0
    assert fb.flop_count("laplacian", 2, 10) == 720
    assert fb.element_matrix_index(3, 4, 2, 3, 0, 0) == 27
    assert fb.element_matrix_index(3, 4, 2, 3, 2, 1) == 32
    assert fb.element_matrix_index(3, 1, 1, 0, 1, 2) == 7
    assert fb.element_matrix_index(3, 1, 1, 2, 0, 0) == 18
    # acceptance.cpp:330-365: the documented decomposition for bs 4, ce 2
    for kr in (3, 4):
        for e in range(8):
            g, r = divmod(e, 4)
            b, z = divmod(r, 2)
            for i in range(kr):
                for j in range(kr):
                    want = g * kr * kr * 4 + b * 2 * kr * kr + z * kr * kr + i + j * kr
                    assert fb.element_matrix_index(kr, 4, 2, e, i, j) == want
    assert fb.store_length("laplacian", 2, 5, 4) == 72
    assert fb.store_length("elasticity", 3, 1, 128) == 128 * 144


@pytest.mark.parametrize("op", list(OPS))
@pytest.mark.parametrize("dim", [2, 3])
def test_analytic_tensor_equals_reference(golden, op, dim):
    assert fb.build_analytic_tensor(op, dim).tobytes() == golden[f"K_{op}_{dim}"].tobytes()


@pytest.mark.parametrize("name,dim,n,jit,seed", [("m2", 2, 4, 0.15, 42), ("m3", 3, 2, 0.15, 42),
                                                 ("m2b", 2, 5, 0.15, 9)])
def test_mesh_synthesis_equals_reference(golden, name, dim, n, jit, seed):
    v, c = fb.structured_mesh(dim, n, jit, seed)
    assert v.tobytes() == golden[f"{name}_vertices"].tobytes()
    assert c.tobytes() == golden[f"{name}_cells"].tobytes()


def test_mesh_synthesis_matches_reference_build_at_scale(reference):
    for dim, n in ((2, 40), (3, 12)):
        v, c = fb.structured_mesh(dim, n, 0.15, 42)
        rv, rc = reference.make_mesh(dim, n, 0.15, 42)
        assert v.tobytes() == rv.tobytes() and c.tobytes() == rc.tobytes()


def test_jitter_validation():
    v, c = fb.structured_mesh(2, 2)
    with pytest.raises(ValueError, match=r"jitter magnitude must lie in \[0, 0.2\]"):
        fb.jitter_mesh(2, v, c, 0.25, 42)


def test_specialize_contract():
    # reference test_engine.cpp:59-85 and kernel_config.cpp:43-55
    with pytest.raises(ValueError, match=r"num_concurrent_elements \(2\) must divide element_batch_size \(5\)"):
        fb.make_variant("laplacian", 3, element_batch_size=5, num_concurrent_elements=2)
    with pytest.raises(ValueError, match="element_batch_size must be positive"):
        fb.make_variant("laplacian", 3, element_batch_size=0)
    with pytest.raises(ValueError, match=r"work-group bound exceeded: krows\^2 \* num_concurrent_elements = 1152 > 1024"):
        fb.make_variant("elasticity", 3, element_batch_size=64, num_concurrent_elements=8)
    fb.make_variant("elasticity", 3, element_batch_size=64, num_concurrent_elements=4)
    with pytest.raises(ValueError, match="analytic tensor was built for a different form"):
        fb.make_variant("elasticity", 3, k=fb.build_analytic_tensor("laplacian", 3))
    assert fb.make_variant("laplacian", 3, "f32", element_batch_size=128, num_concurrent_elements=2,
                           interleave_stores=True).description == "bs128_ce2_is"
    assert fb.make_variant("laplacian", 3, element_batch_size=16, num_concurrent_elements=4,
                           loop_unroll=True).description == "bs16_ce4_unroll"
    assert fb.make_variant("laplacian", 3, element_batch_size=32, interleave_stores=True,
                           loop_unroll=True).description == "bs32_ce1_is_unroll"


@pytest.mark.parametrize("op", list(OPS))
@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_kernel_path_selection(op, dim, prec):
    k = fb.build_analytic_tensor(op, dim)
    assert fb.make_variant(op, dim, prec).path == 3  # reference K: P1 + symmetric + uniform
    broken = k.copy()
    kr = (dim + 1) * dim if op == "elasticity" else dim + 1
    nc = dim + 1 if op == "weighted-laplacian" else 1
    broken[((1 + 1 * kr) * nc) * dim * dim + 1] = 0.5  # off the P1 pattern
    assert fb.make_variant(op, dim, prec, k=broken).path == 2


def test_integration_fails_loudly_without_gpu():
    if fb.device_count() > 0:
        pytest.skip("a GPU is present")
    v, c = fb.structured_mesh(2, 2)
    var = fb.make_variant("laplacian", 2, "f64")
    with pytest.raises(_lib.FembatchError, match="no CUDA device"):
        fb.integrate_mesh(var, v, c)
    with pytest.raises(_lib.FembatchError, match="no CUDA device"):
        fb.pack_geometry(v, c, 2)


def test_validation_precedes_device_use():
    v, c = fb.structured_mesh(2, 2)
    wl = fb.make_variant("weighted-laplacian", 2, "f64")
    with pytest.raises(ValueError, match="form requires a coefficient field"):
        fb.integrate_mesh(wl, v, c)
    lap = fb.make_variant("laplacian", 2, "f64")
    with pytest.raises(ValueError, match="form takes no coefficient field"):
        fb.integrate_mesh(lap, v, c, np.ones(c.size))
    out = np.zeros(5)
    with pytest.raises(ValueError, match="output buffer holds 5 scalars"):
        fb.integrate_mesh(lap, v, c, out=out)


def test_device_alloc_without_a_gpu_fails_loudly():
    import ctypes

    lib = _lib.load()
    err = _lib.fb_error()
    if lib.fb_device_count() == 0:
        assert lib.fb_device_alloc(1024, 0, ctypes.byref(err)) is None
        assert err.code == _lib.FB_ERR_NO_DEVICE
    assert lib.fb_free(None, ctypes.byref(err)) == _lib.FB_OK


def test_host_dtype_checks_without_gpu(fb):
    """Output buffers are never reinterpreted: a wrong-precision numpy `out`
    is rejected before any device work (no GPU needed to reach the check)."""
    import numpy as np
    import pytest

    v, c = fb.structured_mesh(2, 4, 0.0, 42)
    var = fb.make_variant("laplacian", 2, "f32")
    with pytest.raises(fb.engine.L.InvalidArgument, match="out has dtype float64"):
        fb.integrate_mesh(var, v, c, out=np.empty(var.store_length(c.size // 3)))
