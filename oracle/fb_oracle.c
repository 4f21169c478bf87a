/*
 * fb_oracle.c -- TEST INFRASTRUCTURE ONLY (parity checker, never shipped).
 *
 * Plain-C restatement of the reference fembatch arithmetic.  Each function
 * cites the reference file:line it follows (paths relative to
 * /root/reference/proj).  Built with -O2 -ffp-contract=off, exactly like the
 * reference library (src/CMakeLists.txt:16-18), so that every product and
 * sum is individually rounded and the operation order below reproduces the
 * reference bit for bit.  Validated against oracle/_ref (the reference
 * compiled from its own sources) and the golden vectors in tests/golden/.
 */
#include "fb_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* reference.cpp:39-97 -- tabulated symmetric simplex rules, degrees 1..3.   */
int fbo_quadrature(int dim, int degree, double* p, double* w)
{
  if ((dim != 2 && dim != 3) || degree < 1 || degree > 3)
    return FBO_E_ARG;
  if (dim == 2)
  {
    if (degree == 1)
    {
      p[0] = 1.0 / 3.0; p[1] = 1.0 / 3.0;
      w[0] = 1.0 / 2.0;
      return 1;
    }
    if (degree == 2)
    {
      const double pts[6] = {1.0 / 6.0, 1.0 / 6.0, 2.0 / 3.0, 1.0 / 6.0,
                             1.0 / 6.0, 2.0 / 3.0};
      memcpy(p, pts, sizeof pts);
      w[0] = w[1] = w[2] = 1.0 / 6.0;
      return 3;
    }
    {
      const double pts[8] = {1.0 / 3.0, 1.0 / 3.0, 3.0 / 5.0, 1.0 / 5.0,
                             1.0 / 5.0, 3.0 / 5.0, 1.0 / 5.0, 1.0 / 5.0};
      memcpy(p, pts, sizeof pts);
      w[0] = -27.0 / 96.0;
      w[1] = w[2] = w[3] = 25.0 / 96.0;
      return 4;
    }
  }
  if (degree == 1)
  {
    p[0] = p[1] = p[2] = 1.0 / 4.0;
    w[0] = 1.0 / 6.0;
    return 1;
  }
  if (degree == 2)
  {
    const double a = (5.0 - sqrt(5.0)) / 20.0;
    const double b = (5.0 + 3.0 * sqrt(5.0)) / 20.0;
    const double pts[12] = {a, a, a, b, a, a, a, b, a, a, a, b};
    memcpy(p, pts, sizeof pts);
    w[0] = w[1] = w[2] = w[3] = 1.0 / 24.0;
    return 4;
  }
  {
    const double pts[15] = {1.0 / 4.0, 1.0 / 4.0, 1.0 / 4.0, 1.0 / 6.0,
                            1.0 / 6.0, 1.0 / 6.0, 1.0 / 2.0, 1.0 / 6.0,
                            1.0 / 6.0, 1.0 / 6.0, 1.0 / 2.0, 1.0 / 6.0,
                            1.0 / 6.0, 1.0 / 6.0, 1.0 / 2.0};
    memcpy(p, pts, sizeof pts);
    w[0] = -2.0 / 15.0;
    w[1] = w[2] = w[3] = w[4] = 3.0 / 40.0;
    return 5;
  }
}

/* reference.cpp:99-138 -- P1 hat values at a point; gradients are the
 * constant reference gradients: grad phi_0 = (-1,..,-1), grad phi_{d+1} = e_d. */
static void p1_values(int dim, const double* xi, double* v)
{
  double first = 1.0;
  for (int d = 0; d < dim; ++d)
  {
    first -= xi[d];
    v[d + 1] = xi[d];
  }
  v[0] = first;
}

static double p1_grad(int f, int d)
{
  if (f == 0)
    return -1.0;
  return (f - 1 == d) ? 1.0 : 0.0;
}

/* forms.cpp:37-50 */
int fbo_krows(int op, int dim) { return op == 1 ? (dim + 1) * dim : dim + 1; }
int fbo_ncoef(int op, int dim) { return op == 2 ? dim + 1 : 1; }
int64_t fbo_k_len(int op, int dim)
{
  const int64_t kr = fbo_krows(op, dim);
  return kr * kr * fbo_ncoef(op, dim) * dim * dim;
}

/* forms.cpp:52-56 */
static int64_t k_offset(int krows, int ncoef, int dim, int i, int j, int c)
{
  return ((int64_t)(i + j * krows) * ncoef + c) * dim * dim;
}

/* forms.cpp:63-140 specialised to the two jet products the builders use:
 * grad(i) grad(j) [value(c)], summed over the degree-2 rule in point order,
 * each point's product formed left to right starting from 1.0. */
int fbo_build_k(int op, int dim, double* k, int64_t k_len)
{
  if ((dim != 2 && dim != 3) || op < 0 || op > 2)
    return FBO_E_ARG;
  if (k_len != fbo_k_len(op, dim))
    return FBO_E_ARG;
  memset(k, 0, sizeof(double) * (size_t)k_len);
  double pts[15], wts[5];
  const int nq = fbo_quadrature(dim, 2, pts, wts);
  const int nb = dim + 1;
  const int krows = fbo_krows(op, dim);
  const int ncoef = fbo_ncoef(op, dim);

  for (int a = 0; a < nb; ++a)
    for (int b = 0; b < nb; ++b)
      for (int c = 0; c < (op == 2 ? nb : 1); ++c)
        for (int mu = 0; mu < dim; ++mu)
          for (int nu = 0; nu < dim; ++nu)
          {
            double sum = 0.0;
            for (int q = 0; q < nq; ++q)
            {
              double prod = 1.0;
              prod *= p1_grad(a, mu);
              prod *= p1_grad(b, nu);
              if (op == 2)
              {
                double v[4];
                p1_values(dim, pts + q * dim, v);
                prod *= v[c];
              }
              sum += wts[q] * prod;
            }
            if (op == 0)
              k[k_offset(krows, ncoef, dim, a, b, 0) + mu * dim + nu] = sum;
            else if (op == 2)
              k[k_offset(krows, ncoef, dim, a, b, c) + mu * dim + nu] = sum;
            else /* forms.cpp:175-202: 0.25 x scalar jet on c == d blocks */
              for (int comp = 0; comp < dim; ++comp)
                k[k_offset(krows, ncoef, dim, a + comp * nb, b + comp * nb, 0)
                  + mu * dim + nu] = 0.25 * sum;
          }
  return FBO_OK;
}

/* geometry.cpp:27-66 -- edge-vector columns, cofactor determinant,
 * adjugate / det with one IEEE division per entry. */
int fbo_jacobian(int dim, const double* x, double* j, double* jinv,
                 double* det_out)
{
  for (int c = 0; c < dim; ++c)
    for (int r = 0; r < dim; ++r)
      j[r * dim + c] = x[(c + 1) * dim + r] - x[r];
  if (dim == 2)
  {
    const double det = j[0] * j[3] - j[1] * j[2];
    if (!(det > 0.0))
      return 0;
    *det_out = det;
    jinv[0] = j[3] / det;
    jinv[1] = -j[1] / det;
    jinv[2] = -j[2] / det;
    jinv[3] = j[0] / det;
    return 1;
  }
  const double c0 = j[4] * j[8] - j[5] * j[7];
  const double c1 = j[3] * j[8] - j[5] * j[6];
  const double c2 = j[3] * j[7] - j[4] * j[6];
  const double det = j[0] * c0 - j[1] * c1 + j[2] * c2;
  if (!(det > 0.0))
    return 0;
  *det_out = det;
  jinv[0] = (j[4] * j[8] - j[5] * j[7]) / det;
  jinv[1] = (j[2] * j[7] - j[1] * j[8]) / det;
  jinv[2] = (j[1] * j[5] - j[2] * j[4]) / det;
  jinv[3] = (j[5] * j[6] - j[3] * j[8]) / det;
  jinv[4] = (j[0] * j[8] - j[2] * j[6]) / det;
  jinv[5] = (j[2] * j[3] - j[0] * j[5]) / det;
  jinv[6] = (j[3] * j[7] - j[4] * j[6]) / det;
  jinv[7] = (j[1] * j[6] - j[0] * j[7]) / det;
  jinv[8] = (j[0] * j[4] - j[1] * j[3]) / det;
  return 1;
}

/* geometry.cpp:286-302 -- upper triangle, mirrored (bitwise symmetric). */
void fbo_geometry_tensor(int dim, const double* jinv, double det, double* g)
{
  for (int mu = 0; mu < dim; ++mu)
    for (int nu = mu; nu < dim; ++nu)
    {
      double s = 0.0;
      for (int al = 0; al < dim; ++al)
        s += jinv[mu * dim + al] * jinv[nu * dim + al];
      s *= det;
      g[mu * dim + nu] = s;
      g[nu * dim + mu] = s;
    }
}

static int cell_g(int dim, const double* vtx, int64_t nv, const int32_t* cells,
                  int64_t e, double* g)
{
  double x[12], j[9], ji[9], det;
  for (int k = 0; k <= dim; ++k)
  {
    const int32_t v = cells[e * (dim + 1) + k];
    if (v < 0 || v >= nv)
      return FBO_E_RANGE;
    for (int c = 0; c < dim; ++c)
      x[k * dim + c] = vtx[(int64_t)v * dim + c];
  }
  if (!fbo_jacobian(dim, x, j, ji, &det))
    return FBO_E_DEGENERATE;
  fbo_geometry_tensor(dim, ji, det, g);
  return FBO_OK;
}

/* geometry.cpp:312-351 -- slot-major G, padding replicates the last G. */
int fbo_pack_geometry(int dim, const double* vertices, int64_t nv,
                      const int32_t* cells, int64_t ne, int bs, int precision,
                      void* g_out, int64_t* bad_cell)
{
  if ((dim != 2 && dim != 3) || bs < 1)
    return FBO_E_ARG;
  const int dd = dim * dim;
  const int64_t nslots = (ne + bs - 1) / bs * bs;
  double g[9] = {0};
  for (int64_t s = 0; s < nslots; ++s)
  {
    if (s < ne)
    {
      const int rc = cell_g(dim, vertices, nv, cells, s, g);
      if (rc != FBO_OK)
      {
        if (bad_cell)
          *bad_cell = s;
        return rc;
      }
    }
    for (int t = 0; t < dd; ++t)
    {
      if (precision == 0)
        ((float*)g_out)[s * dd + t] = (float)g[t];
      else
        ((double*)g_out)[s * dd + t] = g[t];
    }
  }
  return FBO_OK;
}

/* engine.cpp:37-89 + :91-152 in one precision.  The (k outer, mu, nu)
 * order and the left-associated accumulation from zero are the numerical
 * contract; batch/concurrency/interleave only permute independent writes
 * (store index e*nk + kidx, engine.cpp:130 and :146). */
#define FBO_CONTRACT(S)                                                        \
  static void contract_##S(int op, int dim, const S* g, int64_t nslots,        \
                           int64_t ne, const double* kd, const double* coeffs, \
                           S* out)                                             \
  {                                                                            \
    const int krows = fbo_krows(op, dim);                                      \
    const int nk = krows * krows;                                              \
    const int ncoef = fbo_ncoef(op, dim);                                      \
    const int dd = dim * dim;                                                  \
    const int64_t klen = fbo_k_len(op, dim);                                   \
    S* k = (S*)malloc(sizeof(S) * (size_t)klen);                               \
    for (int64_t t = 0; t < klen; ++t)                                         \
      k[t] = (S)kd[t];                                                         \
    for (int64_t s = 0; s < nslots; ++s)                                       \
    {                                                                          \
      const S* gs = g + s * dd;                                                \
      S w[4] = {0, 0, 0, 0};                                                   \
      if (op == 2)                                                             \
      {                                                                        \
        const int64_t src = s < ne ? s : ne - 1; /* engine.cpp:219-236 */     \
        for (int c = 0; c < ncoef; ++c)                                        \
          w[c] = (S)coeffs[src * ncoef + c];                                   \
      }                                                                        \
      for (int kidx = 0; kidx < nk; ++kidx)                                    \
      {                                                                        \
        const S* kb = k + (int64_t)kidx * ncoef * dd;                          \
        S acc = (S)0;                                                          \
        if (op == 2)                                                           \
        {                                                                      \
          for (int c = 0; c < ncoef; ++c)                                      \
            for (int t = 0; t < dd; ++t)                                       \
              acc += (w[c] * gs[t]) * kb[c * dd + t];                          \
        }                                                                      \
        else                                                                   \
        {                                                                      \
          for (int t = 0; t < dd; ++t)                                         \
            acc += gs[t] * kb[t];                                              \
        }                                                                      \
        out[s * nk + kidx] = acc;                                              \
      }                                                                        \
    }                                                                          \
    free(k);                                                                   \
  }

FBO_CONTRACT(float)
FBO_CONTRACT(double)

int fbo_integrate_packed(int op, int dim, const void* g, int64_t num_batches,
                         int64_t ne, int bs, int precision, const double* k,
                         const double* coeffs, void* out)
{
  if ((dim != 2 && dim != 3) || op < 0 || op > 2 || bs < 1)
    return FBO_E_ARG;
  if (op == 2 && (coeffs == NULL || ne == 0))
    return FBO_E_ARG;
  const int64_t nslots = num_batches * bs;
  if (precision == 0)
    contract_float(op, dim, (const float*)g, nslots, ne, k, coeffs,
                   (float*)out);
  else
    contract_double(op, dim, (const double*)g, nslots, ne, k, coeffs,
                    (double*)out);
  return FBO_OK;
}

int fbo_integrate_mesh(int op, int dim, const double* vertices, int64_t nv,
                       const int32_t* cells, int64_t ne, int bs,
                       int precision, const double* coeffs, void* out,
                       int64_t* bad_cell)
{
  if ((dim != 2 && dim != 3) || bs < 1)
    return FBO_E_ARG;
  const int64_t nb = (ne + bs - 1) / bs;
  const size_t s = precision == 0 ? sizeof(float) : sizeof(double);
  void* g = malloc(s * (size_t)(nb * bs * dim * dim + 1));
  int rc = fbo_pack_geometry(dim, vertices, nv, cells, ne, bs, precision, g,
                             bad_cell);
  if (rc == FBO_OK)
  {
    double* k = (double*)malloc(sizeof(double) * (size_t)fbo_k_len(op, dim));
    fbo_build_k(op, dim, k, fbo_k_len(op, dim));
    rc = fbo_integrate_packed(op, dim, g, nb, ne, bs, precision, k, coeffs,
                              out);
    free(k);
  }
  free(g);
  return rc;
}

/* oracle.cpp:24-109 -- pulled-back gradients per quadrature point, FP64;
 * degree 2 for coefficient-free forms, 3 for the weighted form. */
int fbo_direct(int op, int dim, const double* coords, const double* coeffs,
               double* m)
{
  if ((dim != 2 && dim != 3) || op < 0 || op > 2)
    return FBO_E_ARG;
  double j[9], ji[9], det;
  if (!fbo_jacobian(dim, coords, j, ji, &det))
    return FBO_E_DEGENERATE;
  const int nb = dim + 1;
  const int krows = fbo_krows(op, dim);
  double pts[15], wts[5];
  const int nq = fbo_quadrature(dim, op == 2 ? 3 : 2, pts, wts);
  memset(m, 0, sizeof(double) * (size_t)(krows * krows));
  double pg[4 * 3];
  for (int q = 0; q < nq; ++q)
  {
    for (int f = 0; f < nb; ++f)
      for (int al = 0; al < dim; ++al)
      {
        double s = 0.0;
        for (int mu = 0; mu < dim; ++mu)
          s += ji[mu * dim + al] * p1_grad(f, mu);
        pg[f * dim + al] = s;
      }
    double wq = wts[q] * det;
    if (op == 2)
    {
      double v[4];
      p1_values(dim, pts + q * dim, v);
      double field = 0.0;
      for (int k = 0; k < nb; ++k)
        field += coeffs[k] * v[k];
      wq *= field;
    }
    if (op != 1)
    {
      for (int a = 0; a < nb; ++a)
        for (int b = 0; b < nb; ++b)
        {
          double dot = 0.0;
          for (int al = 0; al < dim; ++al)
            dot += pg[a * dim + al] * pg[b * dim + al];
          m[a * krows + b] += wq * dot;
        }
    }
    else
    {
      for (int c = 0; c < dim; ++c)
        for (int d = 0; d < dim; ++d)
          for (int a = 0; a < nb; ++a)
            for (int b = 0; b < nb; ++b)
            {
              double val = 0.0;
              if (c == d)
              {
                double dot = 0.0;
                for (int al = 0; al < dim; ++al)
                  dot += pg[a * dim + al] * pg[b * dim + al];
                val = 0.25 * dot;
              }
              m[(a + c * nb) * krows + (b + d * nb)] += wq * val;
            }
    }
  }
  return FBO_OK;
}

/* engine.cpp:378-387 */
int64_t fbo_flop_count(int op, int dim, int64_t ne)
{
  const int64_t kr = fbo_krows(op, dim);
  const int64_t nk = kr * kr;
  const int64_t dd = (int64_t)dim * dim;
  if (op != 2)
    return ne * nk * 2 * dd;
  return ne * nk * (dim + 1) * (2 * dd + 2);
}

/* engine.cpp:287-299 */
int64_t fbo_element_matrix_index(int krows, int bs, int ce, int64_t element,
                                 int i, int j)
{
  const int64_t nk = (int64_t)krows * krows;
  const int64_t batch = element / bs;
  const int r = (int)(element % bs);
  return batch * nk * bs + (int64_t)(r / ce) * ce * nk + (int64_t)(r % ce) * nk
         + i + (int64_t)j * krows;
}

/* ------------------------------------------------------------------------
 * Global assembly.  The reference stops at element
 * matrices: global sparse assembly is an explicit non-goal, so
 * there is no reference code to follow.  This is the serial DEFINITION the
 * GPU assembly is checked against:
 *   dof(v, c) = v*nc + c, nc = dim for elasticity (component c of the
 *   reference's local index i = a + c*nb, forms.cpp:175-202) else 1;
 *   pattern = every (dof_i, dof_j) pair of every element, columns sorted;
 *   values: for e = 0..ne-1 ascending, for (i, j):
 *           A[dof_i][dof_j] += Ae[i + j*krows]   (store layout, engine.cpp:287-299)
 *   in engine precision from +0.
 * The pattern is built by sorting all element vertex pairs (independent of
 * the library's vertex-adjacency construction). */
static int cmp_i64(const void* x, const void* y)
{
  const int64_t a = *(const int64_t*)x, b = *(const int64_t*)y;
  return a < b ? -1 : (a > b ? 1 : 0);
}

static int asm_nc(int op, int dim) { return op == 1 ? dim : 1; }

/* Sorted unique vertex pairs va*nv + vb of all elements; *npairs. */
static int64_t* asm_pairs(int dim, const int32_t* cells, int64_t ne, int64_t nv, int64_t* npairs)
{
  const int nb = dim + 1;
  const int64_t n = ne * nb * nb;
  int64_t* p = (int64_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
  if (!p)
    return NULL;
  int64_t k = 0;
  for (int64_t e = 0; e < ne; ++e)
    for (int a = 0; a < nb; ++a)
      for (int b = 0; b < nb; ++b)
        p[k++] = (int64_t)cells[e * nb + a] * nv + cells[e * nb + b];
  qsort(p, (size_t)n, sizeof(int64_t), cmp_i64);
  int64_t u = 0;
  for (int64_t i = 0; i < n; ++i)
    if (u == 0 || p[i] != p[u - 1])
      p[u++] = p[i];
  *npairs = u;
  return p;
}

static int asm_check_cells(int dim, const int32_t* cells, int64_t ne, int64_t nv)
{
  const int nb = dim + 1;
  for (int64_t e = 0; e < ne; ++e)
    for (int a = 0; a < nb; ++a)
    {
      const int32_t v = cells[e * nb + a];
      if (v < 0 || v >= nv)
        return FBO_E_RANGE;
      for (int b = 0; b < a; ++b)
        if (cells[e * nb + b] == v)
          return FBO_E_ARG;
    }
  return FBO_OK;
}

int64_t fbo_assembly_nnz(int op, int dim, const int32_t* cells, int64_t ne, int64_t nv)
{
  if ((dim != 2 && dim != 3) || asm_check_cells(dim, cells, ne, nv) != FBO_OK)
    return -1;
  int64_t np = 0;
  int64_t* p = asm_pairs(dim, cells, ne, nv, &np);
  if (!p)
    return -1;
  free(p);
  const int nc = asm_nc(op, dim);
  return np * nc * nc;
}

int fbo_assembly_pattern(int op, int dim, const int32_t* cells, int64_t ne, int64_t nv,
                         int64_t* row_ptr, int32_t* col_idx)
{
  if (dim != 2 && dim != 3)
    return FBO_E_ARG;
  const int rc = asm_check_cells(dim, cells, ne, nv);
  if (rc != FBO_OK)
    return rc;
  const int nc = asm_nc(op, dim);
  int64_t np = 0;
  int64_t* p = asm_pairs(dim, cells, ne, nv, &np);
  if (!p)
    return FBO_E_ARG;
  /* vertex degree -> row lengths deg*nc for each of the nc rows of a vertex */
  int64_t* first = (int64_t*)calloc((size_t)nv + 1, sizeof(int64_t));
  for (int64_t i = 0; i < np; ++i)
    first[p[i] / nv + 1]++;
  for (int64_t v = 0; v < nv; ++v)
    first[v + 1] += first[v]; /* pair range of vertex v */
  int64_t nz = 0;
  row_ptr[0] = 0;
  for (int64_t v = 0; v < nv; ++v)
    for (int ci = 0; ci < nc; ++ci)
    {
      for (int64_t q = first[v]; q < first[v + 1]; ++q)
        for (int cj = 0; cj < nc; ++cj)
          col_idx[nz++] = (int32_t)((p[q] % nv) * nc + cj);
      row_ptr[v * nc + ci + 1] = nz;
    }
  free(first);
  free(p);
  return FBO_OK;
}

int fbo_assemble(int op, int dim, const int32_t* cells, int64_t ne, int64_t nv, int precision,
                 const void* store, const int64_t* row_ptr, const int32_t* col_idx, void* values)
{
  if (dim != 2 && dim != 3)
    return FBO_E_ARG;
  const int nb = dim + 1, nc = asm_nc(op, dim), kr = nb * nc;
  const int64_t nk = (int64_t)kr * kr, nnz = row_ptr[nv * nc];
  if (precision == 0)
    for (int64_t z = 0; z < nnz; ++z)
      ((float*)values)[z] = 0.0f;
  else
    for (int64_t z = 0; z < nnz; ++z)
      ((double*)values)[z] = 0.0;
  for (int64_t e = 0; e < ne; ++e)
    for (int j = 0; j < kr; ++j)
      for (int i = 0; i < kr; ++i)
      {
        const int64_t row = (int64_t)cells[e * nb + i % nb] * nc + i / nb;
        const int32_t col = (int32_t)((int64_t)cells[e * nb + j % nb] * nc + j / nb);
        int64_t lo = row_ptr[row], hi = row_ptr[row + 1];
        while (lo < hi)
        {
          const int64_t mid = lo + (hi - lo) / 2;
          if (col_idx[mid] < col)
            lo = mid + 1;
          else
            hi = mid;
        }
        if (lo >= row_ptr[row + 1] || col_idx[lo] != col)
          return FBO_E_ARG;
        const int64_t src = e * nk + i + (int64_t)j * kr;
        if (precision == 0)
        {
          float* a = (float*)values + lo;
          *a = *a + ((const float*)store)[src];
        }
        else
        {
          double* a = (double*)values + lo;
          *a = *a + ((const double*)store)[src];
        }
      }
  return FBO_OK;
}
