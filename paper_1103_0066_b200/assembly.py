"""Global CSR assembly from the element-matrix store.

The reference stops at element matrices (global assembly is its declared
non-goal, ``SPEC.md:370``); this is the consumer a finite-element code puts
after ``integrate_mesh``.  ``AssemblyPlan`` wraps the C ABI's
``fb_assembly`` (``include/fembatch_b200.h``, "global assembly"): the CSR
pattern and vertex->element incidence lists are built once per mesh -- on
the GPU for device-resident connectivity and for host meshes of 65,536 or
more elements (uploaded; a CUDA failure there falls back to the host
builder), on the host otherwise or with ``FB_PLAN_HOST=1`` (both builders
give the same plan and the same error for the same bad cell) -- and
``assemble`` runs one deterministic gather kernel on the GPU whose result is
bitwise the serial element-order sum.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L
from .engine import KernelVariant, _as, _chk, _is_torch, _numel, _op, _ptr

FB_ASSEMBLE_SYMMETRIC = 1
FB_ASSEMBLE_BLOCK_DIAGONAL = 2


def _flags(symmetric: bool, block_diagonal: bool) -> int:
    return (FB_ASSEMBLE_SYMMETRIC if symmetric else 0) | (FB_ASSEMBLE_BLOCK_DIAGONAL if block_diagonal else 0)


class AssemblyPlan:
    """CSR plan of the global operator of ``op`` on a mesh's connectivity.

    dof(v, c) = v*nc + c with nc = dim for elasticity, 1 otherwise.
    """

    def __init__(self, op: str, dim: int, cells, num_vertices: int):
        lib = L.load()
        self.op, self.dim = op, dim
        cells = _as(cells, np.int32, "cells")
        self.num_elements = _numel(cells) // (dim + 1)
        self.num_vertices = int(num_vertices)
        err = L.fb_error()
        h = lib.fb_assembly_create(_op(op), dim, _ptr(cells), self.num_elements, self.num_vertices,
                                   C.byref(err))
        if not h:
            L.raise_for(err.code or L.FB_ERR_INVALID_ARGUMENT, err)
        self._h = C.c_void_p(h)
        self._lib = lib

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and h.value:
            self._lib.fb_assembly_free(h)
            self._h = None

    @property
    def rows(self) -> int:
        return self._lib.fb_assembly_rows(self._h)

    @property
    def nnz(self) -> int:
        return self._lib.fb_assembly_nnz(self._h)

    def pattern(self):
        """(row_ptr int64[rows+1], col_idx int32[nnz]) on the host."""
        row_ptr = np.empty(self.rows + 1, dtype=np.int64)
        col_idx = np.empty(self.nnz, dtype=np.int32)
        err = L.fb_error()
        L.raise_for(self._lib.fb_assembly_pattern(self._h, row_ptr.ctypes.data, row_ptr.size,
                                                  col_idx.ctypes.data, col_idx.size, C.byref(err)), err)
        return row_ptr, col_idx

    def assemble(self, variant: KernelVariant, store, values=None, device: int = 0, symmetric: bool = False,
                 block_diagonal: bool = False):
        """CSR values (engine precision) of the element matrices in ``store``.

        ``symmetric=True`` promises bitwise-symmetric element matrices (the
        ``integrate_mesh`` output of a variant with ``path`` 0 or 3): rows are
        then read as contiguous columns.  ``block_diagonal=True`` (elasticity)
        promises element matrices that are zero off the component diagonal
        with bitwise-equal diagonal blocks (``integrate_mesh`` output of any
        variant with ``path`` != 2): only block (0, 0) is read.  The values do
        not depend on either when the promise holds."""
        store = _as(store, variant.dtype, "store")
        if values is None:
            if _is_torch(store) and store.is_cuda:
                import torch
                values = torch.empty(self.nnz, device=store.device,
                                     dtype=torch.float32 if variant.dtype == np.float32 else torch.float64)
            else:
                values = np.empty(self.nnz, dtype=variant.dtype)
        _chk(values, variant.dtype, "values")
        err = L.fb_error()
        rc = self._lib.fb_assemble(self._h, variant.handle, _ptr(store), _numel(store), _ptr(values),
                                   _numel(values), _flags(symmetric, block_diagonal), device,
                                   C.byref(err))
        L.raise_for(rc, err)
        return values

    def assemble_async(self, variant: KernelVariant, store, values, stream: int = 0, symmetric: bool = False,
                       block_diagonal: bool = False):
        """Enqueue the assembly kernel on ``stream`` (device tensors only)."""
        _chk(store, variant.dtype, "store"), _chk(values, variant.dtype, "values")
        err = L.fb_error()
        rc = self._lib.fb_assemble_async(self._h, variant.handle, _ptr(store), _numel(store), _ptr(values),
                                         _numel(values), _flags(symmetric, block_diagonal),
                                         C.c_void_p(stream), C.byref(err))
        L.raise_for(rc, err)

    def assemble_packed(self, variant: KernelVariant, g, coeffs=None, values=None, device: int = 0):
        """CSR values straight from packed geometry ``g`` (host or device; the
        ``integrate_batches`` input): bitwise ``assemble(integrate_batches(g))``
        without ever storing the element matrices."""
        g = _as(g, variant.dtype, "packed geometry")
        coeffs = _as(coeffs, np.float64, "coefficients")
        if values is None:
            if _is_torch(g) and g.is_cuda:
                import torch
                values = torch.empty(self.nnz, device=g.device,
                                     dtype=torch.float32 if variant.dtype == np.float32 else torch.float64)
            else:
                values = np.empty(self.nnz, dtype=variant.dtype)
        _chk(values, variant.dtype, "values")
        err = L.fb_error()
        rc = self._lib.fb_assemble_packed(self._h, variant.handle, _ptr(g), _numel(g), _ptr(coeffs),
                                          _numel(coeffs) if coeffs is not None else 0, _ptr(values),
                                          _numel(values), device, C.byref(err))
        L.raise_for(rc, err)
        return values

    def assemble_packed_async(self, variant: KernelVariant, g, values, coeffs=None, stream: int = 0):
        """Enqueue assembly straight from packed geometry ``g`` (the
        ``integrate_batches`` input, device tensor in engine precision): the
        element matrices are recomputed per incidence and never stored.
        Bitwise ``assemble(integrate_batches(g))``.  Device tensors only."""
        _chk(g, variant.dtype, "packed geometry"), _chk(values, variant.dtype, "values")
        _chk(coeffs, np.float64, "coefficients")
        err = L.fb_error()
        rc = self._lib.fb_assemble_packed_async(self._h, variant.handle, _ptr(g), _numel(g),
                                                _ptr(coeffs) if coeffs is not None else None,
                                                _numel(coeffs) if coeffs is not None else 0,
                                                _ptr(values), _numel(values), C.c_void_p(stream), C.byref(err))
        L.raise_for(rc, err)


def assembly_plan(op: str, dim: int, cells, num_vertices: int) -> AssemblyPlan:
    return AssemblyPlan(op, dim, cells, num_vertices)


def assemble(variant: KernelVariant, plan: AssemblyPlan, store, values=None, device: int = 0,
             symmetric: bool = False):
    return plan.assemble(variant, store, values, device, symmetric)
