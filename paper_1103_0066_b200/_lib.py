"""ctypes binding of libfembatch_b200.so (the C ABI in include/fembatch_b200.h).

The shared library is built in-tree by ``paper_1103_0066_b200.build``; if it is
missing this module raises immediately -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# FB_LIB overrides the library path (same-box A/B experiments only).
LIB_PATH = os.environ.get("FB_LIB") or os.path.join(HERE, "libfembatch_b200.so")

FB_OK, FB_ERR_INVALID_ARGUMENT, FB_ERR_RUNTIME, FB_ERR_OUT_OF_RANGE, FB_ERR_CUDA, FB_ERR_NO_DEVICE = range(6)


class fb_kernel_config(C.Structure):
    _fields_ = [("element_batch_size", C.c_int32), ("num_concurrent_elements", C.c_int32),
                ("interleave_stores", C.c_int32), ("loop_unroll", C.c_int32),
                ("precision", C.c_int32), ("mode", C.c_int32), ("store", C.c_int32),
                ("reserved", C.c_int32)]


class fb_mesh_view(C.Structure):
    _fields_ = [("dim", C.c_int32), ("reserved", C.c_int32), ("num_vertices", C.c_int64),
                ("num_elements", C.c_int64), ("vertices", C.c_void_p), ("cells", C.c_void_p)]


class fb_error(C.Structure):
    _fields_ = [("code", C.c_int32), ("reserved", C.c_int32), ("cell", C.c_int64),
                ("message", C.c_char * 256)]


# name -> (restype, argtypes); every symbol declared in include/fembatch_b200.h
_i32, _i64, _vp = C.c_int, C.c_int64, C.c_void_p
_E = C.POINTER(fb_error)
SIGNATURES = {
    "fb_abi_version": (_i32, []),
    "fb_device_count": (_i32, []),
    "fb_launch_counter": (_i64, []),
    "fb_kernel_setups": (_i64, [_i32]),
    "fb_release_workspace": (_i32, [_i32, _E]),
    "fb_shard_bounds": (_i32, [_i64, _i32, _vp, _E]),
    "fb_krows": (_i32, [_i32, _i32]),
    "fb_k_len": (_i64, [_i32, _i32]),
    "fb_flop_count": (_i64, [_i32, _i32, _i64]),
    "fb_element_matrix_index": (_i64, [_i32, _i32, _i32, _i64, _i32, _i32]),
    "fb_store_length": (_i64, [_i32, _i32, _i64, _i32]),
    "fb_build_analytic_tensor": (_i32, [_i32, _i32, _vp, _i64, _E]),
    "fb_structured_mesh_sizes": (_i32, [_i32, _i32, C.POINTER(_i64), C.POINTER(_i64)]),
    "fb_structured_mesh": (_i32, [_i32, _i32, _vp, _vp, _E]),
    "fb_jitter_mesh": (_i32, [_i32, _vp, _i64, _vp, _i64, C.c_double, C.c_uint64, _E]),
    "fb_specialize": (_vp, [_i32, _i32, _vp, _i64, C.POINTER(fb_kernel_config), _E]),
    "fb_variant_free": (None, [_vp]),
    "fb_variant_description": (C.c_char_p, [_vp]),
    "fb_variant_path": (_i32, [_vp]),
    "fb_integrate_mesh": (_i32, [_vp, C.POINTER(fb_mesh_view), _vp, _vp, _i64, _vp, _i32, _E]),
    "fb_integrate_packed": (_i32, [_vp, _i32, _vp, _i64, _i64, _vp, _vp, _i64, _vp, _i32, _E]),
    "fb_pack_geometry": (_i32, [C.POINTER(fb_mesh_view), _i32, _i32, _vp, _i64, _vp, _i32, _E]),
    "fb_integrate_mesh_async": (_i32, [_vp, C.POINTER(fb_mesh_view), _vp, _vp, _i64, _vp, _vp, _E]),
    "fb_integrate_packed_async": (_i32, [_vp, _i32, _vp, _i64, _i64, _vp, _vp, _i64, _vp, _E]),
    "fb_device_alloc": (_vp, [_i64, _i32, _E]),
    "fb_free": (_i32, [_vp, _E]),
    "fb_pack_geometry_async": (_i32, [C.POINTER(fb_mesh_view), _i32, _i32, _vp, _i64, _vp, _vp, _E]),
    "fb_status_reset": (_i32, [_vp, _vp, _E]),
    "fb_status_check": (_i32, [_vp, _vp, _E]),
    "fb_assembly_create": (_vp, [_i32, _i32, _vp, _i64, _i64, _E]),
    "fb_assembly_free": (None, [_vp]),
    "fb_assembly_rows": (_i64, [_vp]),
    "fb_assembly_nnz": (_i64, [_vp]),
    "fb_assembly_pattern": (_i32, [_vp, _vp, _i64, _vp, _i64, _E]),
    "fb_assemble": (_i32, [_vp, _vp, _vp, _i64, _vp, _i64, _i32, _i32, _E]),
    "fb_assemble_async": (_i32, [_vp, _vp, _vp, _i64, _vp, _i64, _i32, _vp, _E]),
    "fb_assemble_packed_async": (_i32, [_vp, _vp, _vp, _i64, _vp, _i64, _vp, _i64, _vp, _E]),
    "fb_assemble_packed": (_i32, [_vp, _vp, _vp, _i64, _vp, _i64, _vp, _i64, _i32, _E]),
}

_lib = None


def load() -> C.CDLL:
    """Load the in-tree library (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_1103_0066_b200.build` "
            "(there is no CPU fallback for the integration engine)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


class FembatchError(RuntimeError):
    def __init__(self, code: int, message: str, cell: int = -1):
        super().__init__(message)
        self.code = code
        self.cell = cell


class InvalidArgument(FembatchError, ValueError):
    """Reference std::invalid_argument."""


class OutOfRange(FembatchError, IndexError):
    """Reference std::out_of_range."""


class DegenerateElement(FembatchError):
    """Reference std::runtime_error('degenerate element: ...')."""


def raise_for(rc: int, err: fb_error):
    if rc == FB_OK:
        return
    msg = err.message.decode(errors="replace")
    cls = {FB_ERR_INVALID_ARGUMENT: InvalidArgument, FB_ERR_OUT_OF_RANGE: OutOfRange,
           FB_ERR_RUNTIME: DegenerateElement}.get(rc, FembatchError)
    raise cls(rc, msg, int(err.cell))
