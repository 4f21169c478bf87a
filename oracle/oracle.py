"""TEST INFRASTRUCTURE ONLY -- numpy/ctypes front end of the CPU oracle.

Two back ends:

* ``Restatement`` -- ``oracle/liboracle.so``, the plain-C restatement of the
  reference arithmetic (``oracle/fb_oracle.c``; every function cites the
  reference file:line it follows).  Always buildable with gcc.
* ``Reference`` -- ``oracle/_ref/libfembatch_ref.so``, the unmodified reference
  library compiled from ``/root/reference/proj/src`` (``make -C oracle ref``)
  behind the thin ``oracle/ref_shim.cpp``.  Built here; the prebuilt ``.so``
  travels to the GPU box.

Parity is pinned: the restatement is checked against the reference build and
against the reference tests' golden values (``tests/test_oracle.py``).
Nothing in the product path may call this module.
"""
from __future__ import annotations

import ctypes as C
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_RESTATEMENT = os.path.join(HERE, "liboracle.so")
LIB_REFERENCE = os.path.join(HERE, "_ref", "libfembatch_ref.so")

OPS = {"laplacian": 0, "elasticity": 1, "weighted-laplacian": 2}
_i64 = C.c_int64
_i32 = C.c_int
_vp = C.c_void_p
_dp = C.POINTER(C.c_double)


def op_id(op) -> int:
    return OPS[op] if isinstance(op, str) else int(op)


def krows(op, dim: int) -> int:
    return (dim + 1) * dim if op_id(op) == 1 else dim + 1


def ncoef(op, dim: int) -> int:
    return dim + 1 if op_id(op) == 2 else 1


def scalar_dtype(precision) -> np.dtype:
    p = precision if isinstance(precision, int) else {"f32": 0, "f64": 1}[precision]
    return np.dtype(np.float32 if p == 0 else np.float64)


def _prec(precision) -> int:
    return precision if isinstance(precision, int) else {"f32": 0, "f64": 1}[precision]


def _ptr(a):
    return None if a is None else a.ctypes.data_as(_vp)


def build_restatement() -> str:
    """Compile liboracle.so with gcc (used by __graft_entry__.build())."""
    import subprocess

    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)
    return LIB_RESTATEMENT


class OracleError(RuntimeError):
    pass


class Restatement:
    """Plain-C restatement (oracle/fb_oracle.c)."""

    kind = "port"

    def __init__(self, path: str = LIB_RESTATEMENT):
        if not os.path.exists(path):
            build_restatement()
        self.lib = C.CDLL(path)
        L = self.lib
        L.fbo_build_k.argtypes = [_i32, _i32, _vp, _i64]
        L.fbo_jacobian.argtypes = [_i32, _vp, _vp, _vp, _vp]
        L.fbo_geometry_tensor.argtypes = [_i32, _vp, C.c_double, _vp]
        L.fbo_pack_geometry.argtypes = [_i32, _vp, _i64, _vp, _i64, _i32, _i32, _vp, C.POINTER(_i64)]
        L.fbo_integrate_packed.argtypes = [_i32, _i32, _vp, _i64, _i64, _i32, _i32, _vp, _vp, _vp]
        L.fbo_integrate_mesh.argtypes = [_i32, _i32, _vp, _i64, _vp, _i64, _i32, _i32, _vp, _vp, C.POINTER(_i64)]
        L.fbo_direct.argtypes = [_i32, _i32, _vp, _vp, _vp]
        L.fbo_flop_count.argtypes = [_i32, _i32, _i64]
        L.fbo_flop_count.restype = _i64
        L.fbo_element_matrix_index.argtypes = [_i32, _i32, _i32, _i64, _i32, _i32]
        L.fbo_element_matrix_index.restype = _i64
        L.fbo_quadrature.argtypes = [_i32, _i32, _vp, _vp]
        L.fbo_assembly_nnz.argtypes = [_i32, _i32, _vp, _i64, _i64]
        L.fbo_assembly_nnz.restype = _i64
        L.fbo_assembly_pattern.argtypes = [_i32, _i32, _vp, _i64, _i64, _vp, _vp]
        L.fbo_assemble.argtypes = [_i32, _i32, _vp, _i64, _i64, _i32, _vp, _vp, _vp, _vp]

    def quadrature(self, dim, degree):
        p = np.zeros(15)
        w = np.zeros(5)
        n = self.lib.fbo_quadrature(dim, degree, _ptr(p), _ptr(w))
        if n < 0:
            raise OracleError("bad quadrature request")
        return p[: n * dim].reshape(n, dim), w[:n]

    def build_k(self, op, dim) -> np.ndarray:
        n = krows(op, dim) ** 2 * ncoef(op, dim) * dim * dim
        k = np.zeros(n)
        if self.lib.fbo_build_k(op_id(op), dim, _ptr(k), n) != 0:
            raise OracleError("build_k failed")
        return k

    def jacobian(self, dim, coords):
        x = np.ascontiguousarray(coords, dtype=np.float64).ravel()
        j = np.zeros(dim * dim)
        ji = np.zeros(dim * dim)
        det = np.zeros(1)
        ok = self.lib.fbo_jacobian(dim, _ptr(x), _ptr(j), _ptr(ji), _ptr(det))
        if not ok:
            raise OracleError("degenerate element: det(J) <= 0")
        g = np.zeros(dim * dim)
        self.lib.fbo_geometry_tensor(dim, _ptr(ji), float(det[0]), _ptr(g))
        return j, ji, float(det[0]), g

    def pack_geometry(self, vertices, cells, dim, bs, precision):
        v = np.ascontiguousarray(vertices, dtype=np.float64)
        c = np.ascontiguousarray(cells, dtype=np.int32)
        ne = c.size // (dim + 1)
        nslots = -(-ne // bs) * bs
        g = np.zeros(nslots * dim * dim, dtype=scalar_dtype(precision))
        bad = _i64(-1)
        rc = self.lib.fbo_pack_geometry(dim, _ptr(v), v.size // dim, _ptr(c), ne, bs,
                                        _prec(precision), _ptr(g), C.byref(bad))
        if rc != 0:
            raise OracleError(f"degenerate element: det(J) <= 0 in cell {bad.value}")
        return g

    def integrate_packed(self, op, dim, g, ne, bs, precision, k=None, coeffs=None):
        prec = _prec(precision)
        g = np.ascontiguousarray(g, dtype=scalar_dtype(prec))
        nslots = g.size // (dim * dim)
        k = self.build_k(op, dim) if k is None else np.ascontiguousarray(k, dtype=np.float64)
        w = None if coeffs is None else np.ascontiguousarray(coeffs, dtype=np.float64)
        out = np.zeros(nslots * krows(op, dim) ** 2, dtype=scalar_dtype(prec))
        rc = self.lib.fbo_integrate_packed(op_id(op), dim, _ptr(g), nslots // bs, ne, bs, prec,
                                           _ptr(k), _ptr(w), _ptr(out))
        if rc != 0:
            raise OracleError("integrate_packed failed")
        return out

    def integrate_mesh(self, op, vertices, cells, dim, bs=128, precision=1, coeffs=None):
        prec = _prec(precision)
        v = np.ascontiguousarray(vertices, dtype=np.float64)
        c = np.ascontiguousarray(cells, dtype=np.int32)
        ne = c.size // (dim + 1)
        nslots = -(-ne // bs) * bs
        out = np.zeros(nslots * krows(op, dim) ** 2, dtype=scalar_dtype(prec))
        w = None if coeffs is None else np.ascontiguousarray(coeffs, dtype=np.float64)
        bad = _i64(-1)
        rc = self.lib.fbo_integrate_mesh(op_id(op), dim, _ptr(v), v.size // dim, _ptr(c), ne, bs,
                                         prec, _ptr(w), _ptr(out), C.byref(bad))
        if rc == -2:
            raise OracleError(f"degenerate element: det(J) <= 0 in cell {bad.value}")
        if rc != 0:
            raise OracleError(f"integrate_mesh failed ({rc})")
        return out

    def direct(self, op, dim, coords, coeffs=None):
        x = np.ascontiguousarray(coords, dtype=np.float64).ravel()
        w = None if coeffs is None else np.ascontiguousarray(coeffs, dtype=np.float64)
        kr = krows(op, dim)
        m = np.zeros(kr * kr)
        if self.lib.fbo_direct(op_id(op), dim, _ptr(x), _ptr(w), _ptr(m)) != 0:
            raise OracleError("degenerate element")
        return m.reshape(kr, kr)

    def direct_mesh(self, op, vertices, cells, dim, coeffs=None, elements=None):
        """Row-major oracle matrices for the selected elements (FP64)."""
        v = np.asarray(vertices, dtype=np.float64).reshape(-1, dim)
        c = np.asarray(cells, dtype=np.int32).reshape(-1, dim + 1)
        idx = range(c.shape[0]) if elements is None else elements
        w = None if coeffs is None else np.asarray(coeffs, dtype=np.float64).reshape(-1, dim + 1)
        return np.stack([self.direct(op, dim, v[c[e]], None if w is None else w[e]) for e in idx])

    def flop_count(self, op, dim, ne):
        return self.lib.fbo_flop_count(op_id(op), dim, ne)

    def element_matrix_index(self, krows_, bs, ce, e, i, j):
        return self.lib.fbo_element_matrix_index(krows_, bs, ce, e, i, j)

    def assembly_pattern(self, op, dim, cells, nv):
        """CSR pattern (row_ptr int64, col_idx int32) of the global operator."""
        c = np.ascontiguousarray(cells, dtype=np.int32)
        ne = c.size // (dim + 1)
        nnz = self.lib.fbo_assembly_nnz(op_id(op), dim, _ptr(c), ne, nv)
        if nnz < 0:
            raise OracleError("invalid cells for assembly")
        nc = dim if op_id(op) == 1 else 1
        row_ptr = np.zeros(nv * nc + 1, dtype=np.int64)
        col_idx = np.zeros(max(nnz, 1), dtype=np.int32)[:nnz]
        rc = self.lib.fbo_assembly_pattern(op_id(op), dim, _ptr(c), ne, nv, _ptr(row_ptr), _ptr(col_idx))
        if rc != 0:
            raise OracleError(f"assembly_pattern failed ({rc})")
        return row_ptr, col_idx

    def assemble(self, op, dim, cells, nv, precision, store, row_ptr, col_idx):
        """CSR values: element matrices of `store` summed in element order."""
        c = np.ascontiguousarray(cells, dtype=np.int32)
        ne = c.size // (dim + 1)
        s = np.ascontiguousarray(store, dtype=scalar_dtype(precision))
        vals = np.zeros(col_idx.size, dtype=scalar_dtype(precision))
        rc = self.lib.fbo_assemble(op_id(op), dim, _ptr(c), ne, nv, _prec(precision), _ptr(s),
                                   _ptr(row_ptr), _ptr(col_idx), _ptr(vals))
        if rc != 0:
            raise OracleError(f"assemble failed ({rc})")
        return vals


class Reference:
    """The reference library compiled from /root/reference (oracle/_ref)."""

    kind = "reference"

    def __init__(self, path: str = LIB_REFERENCE):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.path = path
        self.lib = C.CDLL(path)
        L = self.lib
        L.ref_last_error.restype = C.c_char_p
        L.ref_mesh_sizes.argtypes = [_i32, _i32, C.POINTER(_i64), C.POINTER(_i64)]
        L.ref_make_mesh.argtypes = [_i32, _i32, C.c_double, C.c_uint64, _vp, _vp]
        L.ref_k_len.argtypes = [_i32, _i32]
        L.ref_k_len.restype = _i64
        L.ref_build_k.argtypes = [_i32, _i32, _vp]
        L.ref_jacobian.argtypes = [_i32, _vp, _vp, _vp, _vp, _vp]
        L.ref_pack_geometry.argtypes = [_i32, _vp, _i64, _vp, _i64, _i32, _i32, _vp]
        L.ref_integrate_mesh.argtypes = [_i32, _i32, _vp, _i64, _vp, _i64, _i32, _i32, _i32, _i32,
                                         _i32, _i32, _vp, _vp]
        L.ref_integrate_packed.argtypes = [_i32, _i32, _vp, _i64, _i64, _i32, _i32, _i32, _vp, _vp]
        L.ref_direct.argtypes = [_i32, _i32, _vp, _vp, _vp]
        L.ref_default_coefficients.argtypes = [_i32, _vp, _i64, _vp, _i64, _vp]
        L.ref_flop_count.argtypes = [_i32, _i32, _i64]
        L.ref_flop_count.restype = _i64
        L.ref_element_matrix_index.argtypes = [_i32, _i32, _i32, _i64, _i32, _i32]
        L.ref_element_matrix_index.restype = _i64
        L.ref_time_integrate.argtypes = [_i32, _i32, _vp, _i64, _vp, _i64, _i32, _i32, _i32, _i32,
                                         _i32, _i32, _i32, _i32, _vp, _dp, _dp]

    def _check(self, rc):
        if rc != 0:
            raise OracleError(self.lib.ref_last_error().decode())

    def write_files(self, op, dim, n, jitter, seed, bs, ce, precision, store_path, mesh_path):
        """The reference's FBEMAT01 store file and text mesh file (golden F4
        fixtures).  Run in a fresh interpreter that has not imported numpy:
        the reference's iostream writers crash inside a numpy process here."""
        import subprocess

        code = ("import ctypes as C, sys\n"
                f"L = C.CDLL({self.path!r})\n"
                "f = L.ref_write_files\n"
                "f.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_uint64, C.c_int, C.c_int, C.c_int,"
                " C.c_char_p, C.c_char_p]\n"
                f"sys.exit(f({op_id(op)}, {dim}, {n}, {float(jitter)!r}, {int(seed)}, {bs}, {ce}, "
                f"{_prec(precision)}, {store_path.encode()!r}, {mesh_path.encode()!r}) != 0)\n")
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True)
        if r.returncode != 0:
            raise OracleError(f"ref_write_files failed: {r.stderr.strip()}")

    def make_mesh(self, dim, n, jitter=0.0, seed=42):
        nv, ne = _i64(), _i64()
        self._check(self.lib.ref_mesh_sizes(dim, n, C.byref(nv), C.byref(ne)))
        v = np.zeros(nv.value * dim)
        c = np.zeros(ne.value * (dim + 1), dtype=np.int32)
        self._check(self.lib.ref_make_mesh(dim, n, jitter, seed, _ptr(v), _ptr(c)))
        return v, c

    def build_k(self, op, dim):
        k = np.zeros(self.lib.ref_k_len(op_id(op), dim))
        self._check(self.lib.ref_build_k(op_id(op), dim, _ptr(k)))
        return k

    def jacobian(self, dim, coords):
        x = np.ascontiguousarray(coords, dtype=np.float64).ravel()
        j, ji, g = np.zeros(dim * dim), np.zeros(dim * dim), np.zeros(dim * dim)
        det = np.zeros(1)
        self._check(self.lib.ref_jacobian(dim, _ptr(x), _ptr(j), _ptr(ji), _ptr(det), _ptr(g)))
        return j, ji, float(det[0]), g

    def pack_geometry(self, vertices, cells, dim, bs, precision):
        v = np.ascontiguousarray(vertices, dtype=np.float64)
        c = np.ascontiguousarray(cells, dtype=np.int32)
        ne = c.size // (dim + 1)
        g = np.zeros(-(-ne // bs) * bs * dim * dim, dtype=scalar_dtype(precision))
        self._check(self.lib.ref_pack_geometry(dim, _ptr(v), v.size // dim, _ptr(c), ne, bs,
                                               _prec(precision), _ptr(g)))
        return g

    def integrate_mesh(self, op, vertices, cells, dim, bs=128, ce=1, interleave=False,
                       unroll=False, precision=1, workers=1, coeffs=None):
        prec = _prec(precision)
        v = np.ascontiguousarray(vertices, dtype=np.float64)
        c = np.ascontiguousarray(cells, dtype=np.int32)
        ne = c.size // (dim + 1)
        out = np.zeros(-(-ne // bs) * bs * krows(op, dim) ** 2, dtype=scalar_dtype(prec))
        w = None if coeffs is None else np.ascontiguousarray(coeffs, dtype=np.float64)
        self._check(self.lib.ref_integrate_mesh(op_id(op), dim, _ptr(v), v.size // dim, _ptr(c), ne,
                                                bs, ce, int(interleave), int(unroll), prec, workers,
                                                _ptr(w), _ptr(out)))
        return out

    def integrate_packed(self, op, dim, g, ne, bs, precision, ce=1, coeffs=None):
        prec = _prec(precision)
        g = np.ascontiguousarray(g, dtype=scalar_dtype(prec))
        nslots = g.size // (dim * dim)
        out = np.zeros(nslots * krows(op, dim) ** 2, dtype=scalar_dtype(prec))
        w = None if coeffs is None else np.ascontiguousarray(coeffs, dtype=np.float64)
        self._check(self.lib.ref_integrate_packed(op_id(op), dim, _ptr(g), nslots // bs, ne, bs, ce,
                                                  prec, _ptr(w), _ptr(out)))
        return out

    def direct(self, op, dim, coords, coeffs=None):
        x = np.ascontiguousarray(coords, dtype=np.float64).ravel()
        w = None if coeffs is None else np.ascontiguousarray(coeffs, dtype=np.float64)
        kr = krows(op, dim)
        m = np.zeros(kr * kr)
        self._check(self.lib.ref_direct(op_id(op), dim, _ptr(x), _ptr(w), _ptr(m)))
        return m.reshape(kr, kr)

    def default_coefficients(self, vertices, cells, dim):
        v = np.ascontiguousarray(vertices, dtype=np.float64)
        c = np.ascontiguousarray(cells, dtype=np.int32)
        ne = c.size // (dim + 1)
        out = np.zeros(ne * (dim + 1))
        self._check(self.lib.ref_default_coefficients(dim, _ptr(v), v.size // dim, _ptr(c), ne,
                                                      _ptr(out)))
        return out

    def flop_count(self, op, dim, ne):
        return self.lib.ref_flop_count(op_id(op), dim, ne)

    def element_matrix_index(self, krows_, bs, ce, e, i, j):
        return self.lib.ref_element_matrix_index(krows_, bs, ce, e, i, j)

    def time_integrate(self, op, vertices, cells, dim, bs=128, ce=2, interleave=True, unroll=False,
                       precision=0, workers=1, reps=3, include_packing=True, coeffs=None):
        v = np.ascontiguousarray(vertices, dtype=np.float64)
        c = np.ascontiguousarray(cells, dtype=np.int32)
        ne = c.size // (dim + 1)
        w = None if coeffs is None else np.ascontiguousarray(coeffs, dtype=np.float64)
        mn, mean = C.c_double(), C.c_double()
        self._check(self.lib.ref_time_integrate(op_id(op), dim, _ptr(v), v.size // dim, _ptr(c), ne,
                                                bs, ce, int(interleave), int(unroll), _prec(precision),
                                                workers, reps, int(include_packing), _ptr(w),
                                                C.byref(mn), C.byref(mean)))
        return mn.value, mean.value


def structured_mesh_numpy(dim: int, n: int):
    """Unjittered structured_simplicial_mesh (reference geometry.cpp:164-234)
    in numpy: vertex (i, j[, k]) / n in lexicographic order; two triangles per
    square / six tetrahedra per cube along the vertex paths (0,..,0) ->
    (1,..,1), odd permutations with vertices 1 and 2 swapped."""
    m = n + 1
    g = np.arange(m, dtype=np.float64) / n
    if dim == 2:
        jj, ii = np.meshgrid(g, g, indexing="ij")
        v = np.stack([ii.ravel(), jj.ravel()], axis=1).ravel()
        j, i = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
        v00 = (i + j * m).ravel()
        v10, v01, v11 = v00 + 1, v00 + m, v00 + m + 1
        c = np.stack([v00, v10, v11, v00, v11, v01], axis=1).reshape(-1, 3)
        return v, np.ascontiguousarray(c.astype(np.int32).ravel())
    kk, jj, ii = np.meshgrid(g, g, g, indexing="ij")
    v = np.stack([ii.ravel(), jj.ravel(), kk.ravel()], axis=1).ravel()
    k, j, i = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
    base = (i + m * (j + m * k)).ravel().astype(np.int64)
    unit = [1, m, m * m]
    perms = [(0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0)]
    odd = [False, True, True, False, False, True]
    tets = []
    for p, o in zip(perms, odd):
        a = base + unit[p[0]]
        b = a + unit[p[1]]
        d = b + unit[p[2]]
        tets.append(np.stack([base, b, a, d] if o else [base, a, b, d], axis=1))
    c = np.stack(tets, axis=1).reshape(-1, 4)
    return v, np.ascontiguousarray(c.astype(np.int32).ravel())


def reference_available() -> bool:
    return os.path.exists(LIB_REFERENCE)


def normwise_error(got: np.ndarray, want: np.ndarray) -> float:
    """Per element max|A-A_o| / max|A_o|, max over elements."""
    got = np.asarray(got, dtype=np.float64).reshape(want.shape[0], -1)
    want = np.asarray(want, dtype=np.float64).reshape(want.shape[0], -1)
    num = np.abs(got - want).max(axis=1)
    den = np.maximum(np.abs(want).max(axis=1), 1e-300)
    return float((num / den).max()) if want.shape[0] else 0.0
