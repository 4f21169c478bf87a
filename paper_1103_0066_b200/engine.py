"""Python front end of the B200 P1 integration engine.

Mirrors the reference operator interface (``/root/reference/proj/include/
fembatch/engine.hpp`` and ``geometry.hpp``): ``make_form_spec`` ->
``build_analytic_tensor`` -> ``specialize_kernel`` -> ``integrate_mesh`` (the
fused ``pack_geometry`` + ``integrate_batches``) or ``pack_geometry`` +
``integrate_batches`` on packed G.  Every integration call goes through the
C ABI into sm_100a kernels; arrays may be numpy (host) or torch CUDA tensors
(device-resident, no copies).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from . import _lib as L

OPERATORS = {"laplacian": 0, "elasticity": 1, "weighted-laplacian": 2}
PRECISIONS = {"f32": 0, "f64": 1}
MODES = {"strict": 0, "fast": 1}
STORES = {"auto": 0, "staged": 1, "direct": 2, "tma": 3}
WORK_GROUP_BOUND = 1024


def _op(op) -> int:
    return OPERATORS[op] if isinstance(op, str) else int(op)


def _prec(p) -> int:
    return PRECISIONS[p] if isinstance(p, str) else int(p)


def scalar_dtype(precision) -> np.dtype:
    return np.dtype(np.float32 if _prec(precision) == 0 else np.float64)


@dataclass(frozen=True)
class FormSpec:
    """Reference FormSpec (include/fembatch/forms.hpp:27-45)."""

    op: str
    dim: int
    num_components: int
    num_basis_funcs: int
    coefficient_arity: int
    geometry_arity: int = 2

    @property
    def krows(self) -> int:
        return self.num_basis_funcs * self.num_components

    @property
    def num_coefficient_blocks(self) -> int:
        return 1 if self.coefficient_arity == 0 else self.num_basis_funcs


def make_form_spec(op: str, dim: int) -> FormSpec:
    if dim not in (2, 3):
        raise L.InvalidArgument(1, f"unsupported spatial dimension {dim}")
    if op not in OPERATORS:
        raise L.InvalidArgument(1, f"unknown operator name: {op}")
    return FormSpec(op, dim, dim if op == "elasticity" else 1, dim + 1,
                    1 if op == "weighted-laplacian" else 0)


def build_analytic_tensor(op: str, dim: int) -> np.ndarray:
    """K in the reference AnalyticTensor layout (forms.cpp:52-56), host precompute."""
    lib = L.load()
    n = lib.fb_k_len(_op(op), dim)
    if n < 0:
        raise L.InvalidArgument(1, f"unsupported form {op} dim={dim}")
    k = np.zeros(n)
    err = L.fb_error()
    L.raise_for(lib.fb_build_analytic_tensor(_op(op), dim, k.ctypes.data, n, C.byref(err)), err)
    return k


@dataclass
class KernelConfig:
    """Reference KernelConfig (kernel_config.hpp:23-37) + GPU mode/store."""

    element_batch_size: int = 128
    num_concurrent_elements: int = 1
    interleave_stores: bool = False
    loop_unroll: bool = False
    precision: str = "f64"
    mode: str = "strict"
    store: str = "auto"

    def to_c(self) -> L.fb_kernel_config:
        return L.fb_kernel_config(self.element_batch_size, self.num_concurrent_elements,
                                  int(self.interleave_stores), int(self.loop_unroll),
                                  _prec(self.precision), MODES[self.mode], STORES[self.store], 0)


class KernelVariant:
    """A frozen device variant (reference KernelVariant, engine.hpp:19-25)."""

    def __init__(self, spec: FormSpec, config: KernelConfig, k: np.ndarray):
        lib = L.load()
        self.spec, self.config = spec, config
        self.k = np.ascontiguousarray(k, dtype=np.float64)
        cfg = config.to_c()
        err = L.fb_error()
        h = lib.fb_specialize(_op(spec.op), spec.dim, self.k.ctypes.data, self.k.size,
                              C.byref(cfg), C.byref(err))
        if not h:
            L.raise_for(err.code or L.FB_ERR_INVALID_ARGUMENT, err)
        self._h = C.c_void_p(h)
        self._lib = lib

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and h.value:
            self._lib.fb_variant_free(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    @property
    def description(self) -> str:
        return self._lib.fb_variant_description(self._h).decode()

    @property
    def path(self) -> int:
        """0 sparse+symmetric, 1 sparse, 2 dense fallback."""
        return self._lib.fb_variant_path(self._h)

    @property
    def dtype(self) -> np.dtype:
        return scalar_dtype(self.config.precision)

    def store_length(self, num_elements: int) -> int:
        bs = self.config.element_batch_size
        return -(-num_elements // bs) * bs * self.spec.krows ** 2


def specialize_kernel(spec: FormSpec, k: np.ndarray, config: KernelConfig) -> KernelVariant:
    return KernelVariant(spec, config, k)


def make_variant(op: str, dim: int, precision: str = "f64", mode: str = "strict",
                 element_batch_size: int = 128, num_concurrent_elements: int = 1,
                 interleave_stores: bool = False, loop_unroll: bool = False,
                 store: str = "auto", k: Optional[np.ndarray] = None) -> KernelVariant:
    spec = make_form_spec(op, dim)
    cfg = KernelConfig(element_batch_size, num_concurrent_elements, interleave_stores, loop_unroll,
                       precision, mode, store)
    return KernelVariant(spec, cfg, build_analytic_tensor(op, dim) if k is None else k)


# ----------------------------------------------------------------- helpers
def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def _ptr(x) -> Optional[int]:
    if x is None:
        return None
    if _is_torch(x):
        if not x.is_contiguous():
            raise L.InvalidArgument(1, "tensor must be contiguous")
        return x.data_ptr()
    if not x.flags["C_CONTIGUOUS"]:
        raise L.InvalidArgument(1, "array must be C-contiguous")
    return x.ctypes.data


def _numel(x) -> int:
    return x.numel() if _is_torch(x) else x.size


def _dtype_name(x) -> str:
    return str(x.dtype).replace("torch.", "")


def _chk(x, dtype, name: str = "array"):
    """Checks (never casts) the element type of an array the C ABI reads or
    writes as raw `dtype` scalars: a torch int64 cells tensor or an f32 store
    passed where f64 is expected would otherwise be reinterpreted."""
    if x is None:
        return x
    want = np.dtype(dtype)
    if _dtype_name(x) != want.name:
        raise L.InvalidArgument(1, f"{name} has dtype {_dtype_name(x)}; {want.name} is required")
    return x


def _as(x, dtype, name: str = "array"):
    """Host arrays are converted to `dtype` (a copy when needed); torch tensors
    are passed through without a copy and must already have it."""
    if x is None:
        return x
    if _is_torch(x):
        return _chk(x, dtype, name)
    return np.ascontiguousarray(x, dtype=dtype)


def _devs(devices: Optional[Sequence[int]]):
    if not devices:
        return None, 0
    arr = (C.c_int * len(devices))(*devices)
    return arr, len(devices)


def mesh_view(vertices, cells, dim: int) -> L.fb_mesh_view:
    return L.fb_mesh_view(dim, 0, _numel(vertices) // dim, _numel(cells) // (dim + 1),
                          _ptr(vertices), _ptr(cells))


def _alloc_out(variant: KernelVariant, n: int, like):
    if like is not None and _is_torch(like) and like.is_cuda:
        import torch
        return torch.empty(n, dtype=torch.float32 if variant.dtype == np.float32 else torch.float64,
                           device=like.device)
    return np.empty(n, dtype=variant.dtype)


# ------------------------------------------------------------- integration
def integrate_mesh(variant: KernelVariant, vertices, cells, coefficients=None, out=None,
                   devices: Optional[Sequence[int]] = None):
    """Mesh + form in, every element matrix out (fused pack_geometry + integrate_batches).

    Returns the reference ElementMatrixStore scalars (length
    ``variant.store_length(num_elements)``, element-major, ``e*krows^2 + i + j*krows``).
    """
    lib = L.load()
    dim = variant.spec.dim
    vertices, cells = _as(vertices, np.float64, "vertices"), _as(cells, np.int32, "cells")
    coefficients = _as(coefficients, np.float64, "coefficients")
    ne = _numel(cells) // (dim + 1)
    n = variant.store_length(ne)
    if out is None:
        out = _alloc_out(variant, n, cells)
    _chk(out, variant.dtype, "out")
    mv = mesh_view(vertices, cells, dim)
    dv, nd = _devs(devices)
    err = L.fb_error()
    rc = lib.fb_integrate_mesh(variant.handle, C.byref(mv), _ptr(coefficients), _ptr(out),
                               _numel(out), dv, nd, C.byref(err))
    L.raise_for(rc, err)
    return out


def integrate_batches(variant: KernelVariant, g, num_elements: int, coefficients=None, out=None,
                      devices: Optional[Sequence[int]] = None):
    """Reference integrate_batches on packed G (slot-major, engine precision)."""
    lib = L.load()
    dim = variant.spec.dim
    g = _as(g, variant.dtype, "packed geometry")
    coefficients = _as(coefficients, np.float64, "coefficients")
    bs = variant.config.element_batch_size
    nslots = _numel(g) // (dim * dim)
    if nslots % bs:
        raise L.InvalidArgument(1, "geometry was packed for a different batch size")
    n = nslots * variant.spec.krows ** 2
    if out is None:
        out = _alloc_out(variant, n, g)
    _chk(out, variant.dtype, "out")
    dv, nd = _devs(devices)
    err = L.fb_error()
    rc = lib.fb_integrate_packed(variant.handle, dim, _ptr(g), nslots // bs, num_elements,
                                 _ptr(coefficients), _ptr(out), _numel(out), dv, nd, C.byref(err))
    L.raise_for(rc, err)
    return out


def pack_geometry(vertices, cells, dim: int, element_batch_size: int = 128,
                  precision: str = "f64", out=None, devices: Optional[Sequence[int]] = None):
    """GPU pack_geometry: G in the reference PackedGeometry layout."""
    lib = L.load()
    vertices, cells = _as(vertices, np.float64, "vertices"), _as(cells, np.int32, "cells")
    ne = _numel(cells) // (dim + 1)
    n = -(-ne // element_batch_size) * element_batch_size * dim * dim
    if out is None:
        if _is_torch(cells) and cells.is_cuda:
            import torch
            out = torch.empty(n, dtype=torch.float32 if _prec(precision) == 0 else torch.float64,
                              device=cells.device)
        else:
            out = np.empty(n, dtype=scalar_dtype(precision))
    _chk(out, scalar_dtype(precision), "out")
    mv = mesh_view(vertices, cells, dim)
    dv, nd = _devs(devices)
    err = L.fb_error()
    rc = lib.fb_pack_geometry(C.byref(mv), element_batch_size, _prec(precision), _ptr(out),
                              _numel(out), dv, nd, C.byref(err))
    L.raise_for(rc, err)
    return out


def integrate_mesh_async(variant: KernelVariant, vertices, cells, out, status, stream: int = 0,
                         coefficients=None):
    """Enqueue the fused kernel on ``stream`` (device tensors only; no sync)."""
    lib = L.load()
    _chk(vertices, np.float64, "vertices"), _chk(cells, np.int32, "cells")
    _chk(coefficients, np.float64, "coefficients"), _chk(out, variant.dtype, "out")
    _chk(status, np.int64, "status")
    mv = mesh_view(vertices, cells, variant.spec.dim)
    err = L.fb_error()
    rc = lib.fb_integrate_mesh_async(variant.handle, C.byref(mv), _ptr(coefficients), _ptr(out),
                                     _numel(out), _ptr(status), C.c_void_p(stream), C.byref(err))
    L.raise_for(rc, err)


def integrate_packed_async(variant: KernelVariant, g, num_elements: int, out, stream: int = 0,
                           coefficients=None):
    lib = L.load()
    dim = variant.spec.dim
    _chk(g, variant.dtype, "packed geometry"), _chk(out, variant.dtype, "out")
    _chk(coefficients, np.float64, "coefficients")
    nslots = _numel(g) // (dim * dim)
    err = L.fb_error()
    rc = lib.fb_integrate_packed_async(variant.handle, dim, _ptr(g),
                                       nslots // variant.config.element_batch_size, num_elements,
                                       _ptr(coefficients), _ptr(out), _numel(out),
                                       C.c_void_p(stream), C.byref(err))
    L.raise_for(rc, err)


def pack_geometry_async(vertices, cells, dim: int, g_out, status, element_batch_size: int = 128,
                        precision: str = "f64", stream: int = 0):
    """Enqueue the GPU pack_geometry kernel on ``stream`` (device tensors only)."""
    _chk(vertices, np.float64, "vertices"), _chk(cells, np.int32, "cells")
    _chk(g_out, scalar_dtype(precision), "g_out"), _chk(status, np.int64, "status")
    mv = mesh_view(vertices, cells, dim)
    err = L.fb_error()
    rc = L.load().fb_pack_geometry_async(C.byref(mv), element_batch_size, _prec(precision), _ptr(g_out),
                                         _numel(g_out), _ptr(status), C.c_void_p(stream), C.byref(err))
    L.raise_for(rc, err)


def status_reset(status, stream: int = 0):
    _chk(status, np.int64, "status")
    err = L.fb_error()
    L.raise_for(L.load().fb_status_reset(_ptr(status), C.c_void_p(stream), C.byref(err)), err)


def status_check(status, stream: int = 0):
    _chk(status, np.int64, "status")
    err = L.fb_error()
    L.raise_for(L.load().fb_status_check(_ptr(status), C.c_void_p(stream), C.byref(err)), err)


# ------------------------------------------------------------ pure helpers
def flop_count(op: str, dim: int, num_elements: int) -> int:
    return L.load().fb_flop_count(_op(op), dim, num_elements)


def element_matrix_index(krows: int, bs: int, ce: int, element: int, i: int, j: int) -> int:
    return L.load().fb_element_matrix_index(krows, bs, ce, element, i, j)


def store_length(op: str, dim: int, num_elements: int, bs: int) -> int:
    return L.load().fb_store_length(_op(op), dim, num_elements, bs)


def unpack_element_matrix(store, krows: int, element: int) -> np.ndarray:
    """Row-major krows x krows matrix of one element (reference engine.cpp:389-411)."""
    s = store.cpu().numpy() if _is_torch(store) else store
    base = element * krows * krows
    return np.asarray(s[base:base + krows * krows], dtype=np.float64).reshape(krows, krows).T.copy()


def launch_counter() -> int:
    return L.load().fb_launch_counter()


def device_count() -> int:
    return L.load().fb_device_count()


def kernel_setups(device: int) -> int:
    """Per-device kernel setups (shared-memory opt-in + occupancy) so far."""
    return L.load().fb_kernel_setups(device)


def release_workspace(device: int = -1) -> None:
    """Free the library's staging workspace and streams on ``device`` (-1: all)."""
    err = L.fb_error()
    L.raise_for(L.load().fb_release_workspace(device, C.byref(err)), err)


def shard_bounds(num_slots: int, parts: int) -> list:
    """The engine's element-range split for a device list (fb_shard_bounds):
    ``[b_0 = 0, ..., b_parts = num_slots]``, contiguous and tile aligned; shard g
    integrates slots ``[b_g, b_g+1)`` and its output is that slice of the store."""
    b = (C.c_int64 * (max(parts, 0) + 1))()
    err = L.fb_error()
    L.raise_for(L.load().fb_shard_bounds(num_slots, parts, b, C.byref(err)), err)
    return list(b)
