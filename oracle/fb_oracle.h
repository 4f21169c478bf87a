/*
 * fb_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C CPU restatement of the reference fembatch hot path
 * (/root/reference/proj/src/{geometry,forms,reference,engine,oracle}.cpp),
 * used as the parity checker for the CUDA engine.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it.
 * The product library (paper_1103_0066_b200/) never links or calls this.
 *
 * Parity of this restatement is pinned against the reference compiled from
 * its own sources (oracle/_ref, see oracle/Makefile) and against the
 * reference tests' hand-written golden values (tests/golden/).
 *
 * Operators: 0 = laplacian, 1 = elasticity, 2 = weighted-laplacian.
 * Precision: 0 = f32, 1 = f64.
 * Return codes: 0 ok, <0 error (see FBO_E_*).
 */
#ifndef FB_ORACLE_H
#define FB_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FBO_OK 0
#define FBO_E_ARG (-1)
#define FBO_E_DEGENERATE (-2)
#define FBO_E_RANGE (-3)

/* reference.cpp:39-97 -- returns number of points, or <0. */
int fbo_quadrature(int dim, int degree, double* points, double* weights);

/* forms.cpp:37-50 shape helpers. */
int fbo_krows(int op, int dim);
int fbo_ncoef(int op, int dim);
int64_t fbo_k_len(int op, int dim);

/* forms.cpp:63-246 -- K in AnalyticTensor layout. */
int fbo_build_k(int op, int dim, double* k, int64_t k_len);

/* geometry.cpp:27-66 -- returns 1 if det > 0, 0 otherwise. */
int fbo_jacobian(int dim, const double* x, double* j, double* jinv,
                 double* det);

/* geometry.cpp:286-302 */
void fbo_geometry_tensor(int dim, const double* jinv, double det, double* g);

/* geometry.cpp:312-351 -- G in PackedGeometry layout (num_batches*bs*dim^2
 * scalars of the requested precision).  *bad_cell receives the first
 * degenerate cell on FBO_E_DEGENERATE. */
int fbo_pack_geometry(int dim, const double* vertices, int64_t nv,
                      const int32_t* cells, int64_t ne, int bs,
                      int precision, void* g_out, int64_t* bad_cell);

/* engine.cpp:91-152 + :194-283 -- contraction of packed G with K cast to
 * engine precision; store layout e*nk + i + j*krows over num_batches*bs
 * slots.  coeffs: ne*nb doubles (weighted form only, else NULL). */
int fbo_integrate_packed(int op, int dim, const void* g, int64_t num_batches,
                         int64_t ne, int bs, int precision, const double* k,
                         const double* coeffs, void* out);

/* pack + integrate composition (tests/test_engine.cpp:28-38). */
int fbo_integrate_mesh(int op, int dim, const double* vertices, int64_t nv,
                       const int32_t* cells, int64_t ne, int bs,
                       int precision, const double* coeffs, void* out,
                       int64_t* bad_cell);

/* oracle.cpp:24-109 -- direct physical-space quadrature, FP64, row-major
 * krows x krows. */
int fbo_direct(int op, int dim, const double* coords, const double* coeffs,
               double* m);

/* engine.cpp:378-387 */
int64_t fbo_flop_count(int op, int dim, int64_t ne);

/* engine.cpp:287-299 */
int64_t fbo_element_matrix_index(int krows, int bs, int ce, int64_t element,
                                 int i, int j);

/* Global assembly (no reference counterpart: SPEC.md:370 non-goal; the
 * serial definition the GPU assembly is checked against).  dof = v*nc + c,
 * nc = dim for elasticity else 1; CSR with sorted columns; values summed in
 * ascending element order in engine precision from +0. */
int64_t fbo_assembly_nnz(int op, int dim, const int32_t* cells, int64_t ne, int64_t nv);
int fbo_assembly_pattern(int op, int dim, const int32_t* cells, int64_t ne, int64_t nv,
                         int64_t* row_ptr, int32_t* col_idx);
int fbo_assemble(int op, int dim, const int32_t* cells, int64_t ne, int64_t nv, int precision,
                 const void* store, const int64_t* row_ptr, const int32_t* col_idx, void* values);

#ifdef __cplusplus
}
#endif

#endif
