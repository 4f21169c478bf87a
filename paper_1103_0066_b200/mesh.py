"""Input synthesis: the reference's structured / jittered simplicial meshes.

Bit-identical to ``structured_simplicial_mesh`` + ``jitter_mesh``
(reference src/geometry.cpp:164-262), implemented natively in the engine
library (csrc/fb_host.cpp) so benchmarks and tests can build the reference's
inputs on a box that does not have the reference.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L


def structured_mesh_sizes(dim: int, n: int):
    nv, ne = C.c_int64(), C.c_int64()
    if L.load().fb_structured_mesh_sizes(dim, n, C.byref(nv), C.byref(ne)) != 0:
        raise L.InvalidArgument(1, f"bad structured mesh request dim={dim} n={n}")
    return nv.value, ne.value


def structured_mesh(dim: int, n: int, jitter: float = 0.0, seed: int = 42):
    """(vertices float64[nv*dim], cells int32[ne*(dim+1)])."""
    lib = L.load()
    nv, ne = structured_mesh_sizes(dim, n)
    v = np.empty(nv * dim, dtype=np.float64)
    c = np.empty(ne * (dim + 1), dtype=np.int32)
    err = L.fb_error()
    L.raise_for(lib.fb_structured_mesh(dim, n, v.ctypes.data, c.ctypes.data, C.byref(err)), err)
    if jitter > 0.0:
        jitter_mesh(dim, v, c, jitter, seed)
    return v, c


def jitter_mesh(dim: int, vertices: np.ndarray, cells: np.ndarray, magnitude: float, seed: int):
    """In place (reference jitter_mesh semantics)."""
    assert vertices.dtype == np.float64 and cells.dtype == np.int32
    err = L.fb_error()
    rc = L.load().fb_jitter_mesh(dim, vertices.ctypes.data, vertices.size // dim, cells.ctypes.data,
                                 cells.size // (dim + 1), float(magnitude), int(seed), C.byref(err))
    L.raise_for(rc, err)
    return vertices


def resolution_for(dim: int, num_elements: int) -> int:
    """Smallest n whose structured mesh has >= num_elements cells."""
    n = 1
    while structured_mesh_sizes(dim, n)[1] < num_elements:
        n += 1
    return n


def mesh_prefix(dim: int, num_elements: int, jitter: float = 0.0, seed: int = 42):
    """The first ``num_elements`` cells of the smallest structured mesh that has
    them (a contiguous slab with exact power-of-two
    counts).  The vertex array is kept whole."""
    n = resolution_for(dim, num_elements)
    v, c = structured_mesh(dim, n, jitter, seed)
    return v, np.ascontiguousarray(c[: num_elements * (dim + 1)]), n
