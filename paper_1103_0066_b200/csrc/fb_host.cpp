// fb_host.cpp -- see fb_host.h.  Compiled with -ffp-contract=off so every
// product and sum rounds individually, as in the reference build
// (src/CMakeLists.txt:16-18); K and the jittered coordinates then come out
// bitwise identical to the reference's.
#include "fb_host.h"

#include <algorithm>
#include <cmath>
#include <limits>
#include <random>
#include <stdexcept>
#include <string>

namespace fbh {

void check_dim(int dim)
{
  if (dim != 2 && dim != 3)
    throw std::invalid_argument("unsupported spatial dimension " + std::to_string(dim));
}

static void check_op(int op)
{
  if (op < 0 || op > 2)
    throw std::invalid_argument("unknown operator");
}

int krows(int op, int dim) { return op == 1 ? (dim + 1) * dim : dim + 1; }
int ncoef(int op, int dim) { return op == 2 ? dim + 1 : 1; }
int64_t k_len(int op, int dim)
{
  const int64_t kr = krows(op, dim);
  return kr * kr * ncoef(op, dim) * dim * dim;
}

// Symmetric simplex rules, reference src/reference.cpp:39-97.
void quadrature(int dim, int degree, std::vector<double>& p, std::vector<double>& w)
{
  check_dim(dim);
  if (degree < 1 || degree > 3)
    throw std::invalid_argument("no tabulated simplex rule for degree " + std::to_string(degree));
  if (dim == 2)
  {
    switch (degree)
    {
    case 1:
      p = {1.0 / 3.0, 1.0 / 3.0};
      w = {0.5};
      return;
    case 2:
      p = {1.0 / 6.0, 1.0 / 6.0, 2.0 / 3.0, 1.0 / 6.0, 1.0 / 6.0, 2.0 / 3.0};
      w.assign(3, 1.0 / 6.0);
      return;
    default:
      p = {1.0 / 3.0, 1.0 / 3.0, 0.6, 0.2, 0.2, 0.6, 0.2, 0.2};
      w = {-27.0 / 96.0, 25.0 / 96.0, 25.0 / 96.0, 25.0 / 96.0};
      return;
    }
  }
  switch (degree)
  {
  case 1:
    p.assign(3, 0.25);
    w = {1.0 / 6.0};
    return;
  case 2:
  {
    const double lo = (5.0 - std::sqrt(5.0)) / 20.0;
    const double hi = (5.0 + 3.0 * std::sqrt(5.0)) / 20.0;
    p = {lo, lo, lo, hi, lo, lo, lo, hi, lo, lo, lo, hi};
    w.assign(4, 1.0 / 24.0);
    return;
  }
  default:
  {
    const double s = 1.0 / 6.0;
    p = {0.25, 0.25, 0.25, s, s, s, 0.5, s, s, s, 0.5, s, s, s, 0.5};
    w = {-2.0 / 15.0, 3.0 / 40.0, 3.0 / 40.0, 3.0 / 40.0, 3.0 / 40.0};
    return;
  }
  }
}

namespace {

// Reference-space P1 gradient component: grad phi_0 = -1, grad phi_{d+1} = e_d.
double grad(int f, int d) { return f == 0 ? -1.0 : (f - 1 == d ? 1.0 : 0.0); }

// Barycentric value phi_f at point xi (reference.cpp:108-118 ordering).
double value(int dim, int f, const double* xi)
{
  if (f > 0)
    return xi[f - 1];
  double first = 1.0;
  for (int d = 0; d < dim; ++d)
    first -= xi[d];
  return first;
}

}  // namespace

// Exact quadrature of the jet products grad(a) grad(b) [value(c)] with the
// degree-2 rule (forms.cpp:63-140, builders :155-232): per point the product
// is formed left to right from 1.0, then accumulated w_q * product from 0.
std::vector<double> build_analytic_tensor(int op, int dim)
{
  check_op(op);
  check_dim(dim);
  std::vector<double> pts, wts;
  quadrature(dim, 2, pts, wts);
  const int nb = dim + 1;
  const int kr = krows(op, dim);
  const int nc = ncoef(op, dim);
  const int dd = dim * dim;
  std::vector<double> k(static_cast<size_t>(k_len(op, dim)), 0.0);
  auto at = [&](int i, int j, int c, int t) -> double&
  { return k[static_cast<size_t>((static_cast<int64_t>(i + j * kr) * nc + c) * dd + t)]; };

  for (int a = 0; a < nb; ++a)
    for (int b = 0; b < nb; ++b)
      for (int c = 0; c < nc; ++c)
        for (int mu = 0; mu < dim; ++mu)
          for (int nu = 0; nu < dim; ++nu)
          {
            double acc = 0.0;
            for (size_t q = 0; q < wts.size(); ++q)
            {
              double prod = 1.0 * grad(a, mu);
              prod = prod * grad(b, nu);
              if (op == 2)
                prod = prod * value(dim, c, &pts[q * dim]);
              acc = acc + wts[q] * prod;
            }
            if (op != 1)
              at(a, b, c, mu * dim + nu) = acc;
            else  // vector basis phi_a e_comp: only comp == comp' blocks, scaled by 1/4
              for (int comp = 0; comp < dim; ++comp)
                at(a + comp * nb, b + comp * nb, 0, mu * dim + nu) = 0.25 * acc;
          }
  return k;
}

void structured_mesh_sizes(int dim, int n, int64_t& nv, int64_t& ne)
{
  check_dim(dim);
  if (n < 1)
    throw std::invalid_argument("mesh resolution must be >= 1");
  const int64_t m = n + 1;
  nv = dim == 2 ? m * m : m * m * m;
  ne = dim == 2 ? 2 * static_cast<int64_t>(n) * n : 6 * static_cast<int64_t>(n) * n * n;
}

// src/geometry.cpp:164-234: lexicographic vertices (x fastest) at i/n; two
// triangles per square, six path tetrahedra per cube with odd permutations
// swapped to stay positively oriented.
void structured_mesh(int dim, int n, double* v, int32_t* cells)
{
  int64_t nv, ne;
  structured_mesh_sizes(dim, n, nv, ne);
  const int64_t m = n + 1;
  if (dim == 2)
  {
    for (int64_t j = 0; j < m; ++j)
      for (int64_t i = 0; i < m; ++i)
      {
        v[2 * (i + j * m)] = static_cast<double>(i) / n;
        v[2 * (i + j * m) + 1] = static_cast<double>(j) / n;
      }
    int32_t* c = cells;
    for (int64_t j = 0; j < n; ++j)
      for (int64_t i = 0; i < n; ++i)
      {
        const int32_t a = static_cast<int32_t>(i + j * m), b = a + 1;
        const int32_t d = static_cast<int32_t>(a + m), e = d + 1;
        const int32_t tri[6] = {a, b, e, a, e, d};
        std::copy(tri, tri + 6, c);
        c += 6;
      }
    return;
  }
  for (int64_t k = 0; k < m; ++k)
    for (int64_t j = 0; j < m; ++j)
      for (int64_t i = 0; i < m; ++i)
      {
        double* p = v + 3 * (i + m * (j + m * k));
        p[0] = static_cast<double>(i) / n;
        p[1] = static_cast<double>(j) / n;
        p[2] = static_cast<double>(k) / n;
      }
  static const int order[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
  static const bool flip[6] = {false, true, true, false, false, true};
  int32_t* c = cells;
  for (int64_t k = 0; k < n; ++k)
    for (int64_t j = 0; j < n; ++j)
      for (int64_t i = 0; i < n; ++i)
        for (int p = 0; p < 6; ++p)
        {
          int64_t at[3] = {i, j, k};
          c[0] = static_cast<int32_t>(i + m * (j + m * k));
          for (int s = 0; s < 3; ++s)
          {
            at[order[p][s]] += 1;
            c[s + 1] = static_cast<int32_t>(at[0] + m * (at[1] + m * at[2]));
          }
          if (flip[p])
            std::swap(c[1], c[2]);
          c += 4;
        }
}

namespace {

// Vertices on a facet owned by exactly one cell.  Facets are bucketed by
// their smallest vertex (counting sort), then matched inside each bucket.
std::vector<char> boundary_vertices(int dim, int64_t nv, const int32_t* cells, int64_t ne)
{
  const int nb = dim + 1;
  std::vector<int64_t> start(static_cast<size_t>(nv) + 1, 0);
  auto facet = [&](int64_t e, int omit, int32_t (&f)[3])
  {
    int len = 0;
    for (int k = 0; k < nb; ++k)
      if (k != omit)
        f[len++] = cells[e * nb + k];
    std::sort(f, f + len);
    if (len == 2)
      f[2] = -1;
  };
  for (int64_t e = 0; e < ne; ++e)
    for (int omit = 0; omit < nb; ++omit)
    {
      int32_t f[3];
      facet(e, omit, f);
      ++start[static_cast<size_t>(f[0]) + 1];
    }
  for (int64_t v = 0; v < nv; ++v)
    start[v + 1] += start[v];
  std::vector<int64_t> fill(start.begin(), start.end() - 1);
  std::vector<uint64_t> rest(static_cast<size_t>(ne) * nb);  // (f1, f2) packed
  for (int64_t e = 0; e < ne; ++e)
    for (int omit = 0; omit < nb; ++omit)
    {
      int32_t f[3];
      facet(e, omit, f);
      rest[static_cast<size_t>(fill[f[0]]++)]
          = (static_cast<uint64_t>(static_cast<uint32_t>(f[1])) << 32) | static_cast<uint32_t>(f[2]);
    }
  std::vector<char> boundary(static_cast<size_t>(nv), 0);
  for (int64_t v = 0; v < nv; ++v)
  {
    auto b = rest.begin() + start[v], e = rest.begin() + start[v + 1];
    std::sort(b, e);
    for (auto it = b; it != e;)
    {
      auto run = it;
      while (run != e && *run == *it)
        ++run;
      if (run - it == 1)
      {
        boundary[static_cast<size_t>(v)] = 1;
        boundary[static_cast<size_t>(*it >> 32)] = 1;
        if (dim == 3)
          boundary[static_cast<size_t>(*it & 0xffffffffu)] = 1;
      }
      it = run;
    }
  }
  return boundary;
}

}  // namespace

// src/geometry.cpp:236-262: interior vertices move by (2u-1)*magnitude*h per
// coordinate, u from mt19937_64 (53-bit mantissa mapping), h = shortest
// incident edge; one draw per (vertex, coordinate), boundary included.
void jitter_mesh(int dim, double* v, int64_t nv, const int32_t* cells, int64_t ne,
                 double magnitude, uint64_t seed)
{
  check_dim(dim);
  if (!(magnitude >= 0.0) || magnitude > 0.2)
    throw std::invalid_argument("jitter magnitude must lie in [0, 0.2]");
  for (int64_t t = 0; t < ne * (dim + 1); ++t)
    if (cells[t] < 0 || cells[t] >= nv)
      throw std::invalid_argument("cell vertex index " + std::to_string(cells[t]) + " out of range");
  const std::vector<char> boundary = boundary_vertices(dim, nv, cells, ne);
  std::vector<double> h(static_cast<size_t>(nv), std::numeric_limits<double>::infinity());
  const int nb = dim + 1;
  for (int64_t e = 0; e < ne; ++e)
    for (int a = 0; a < nb; ++a)
      for (int b = a + 1; b < nb; ++b)
      {
        const int32_t va = cells[e * nb + a], vb = cells[e * nb + b];
        double len2 = 0.0;
        for (int c = 0; c < dim; ++c)
        {
          const double d = v[static_cast<int64_t>(va) * dim + c] - v[static_cast<int64_t>(vb) * dim + c];
          len2 = len2 + d * d;
        }
        const double len = std::sqrt(len2);
        h[va] = std::min(h[va], len);
        h[vb] = std::min(h[vb], len);
      }
  std::mt19937_64 rng(seed);
  for (int64_t i = 0; i < nv; ++i)
    for (int c = 0; c < dim; ++c)
    {
      const double u = static_cast<double>(rng() >> 11) * 0x1.0p-53;
      if (!boundary[static_cast<size_t>(i)])
        v[i * dim + c] += (2.0 * u - 1.0) * magnitude * h[static_cast<size_t>(i)];
    }
  check_cells(dim, v, nv, cells, ne);
}

bool jacobian(int dim, const double* x, double* j, double* ji, double* det_out)
{
  for (int c = 0; c < dim; ++c)
    for (int r = 0; r < dim; ++r)
      j[r * dim + c] = x[(c + 1) * dim + r] - x[r];
  double det;
  if (dim == 2)
  {
    det = j[0] * j[3] - j[1] * j[2];
    ji[0] = j[3] / det;
    ji[1] = -j[1] / det;
    ji[2] = -j[2] / det;
    ji[3] = j[0] / det;
  }
  else
  {
    const double m0 = j[4] * j[8] - j[5] * j[7];
    const double m1 = j[3] * j[8] - j[5] * j[6];
    const double m2 = j[3] * j[7] - j[4] * j[6];
    det = j[0] * m0 - j[1] * m1 + j[2] * m2;
    ji[0] = m0 / det;
    ji[1] = (j[2] * j[7] - j[1] * j[8]) / det;
    ji[2] = (j[1] * j[5] - j[2] * j[4]) / det;
    ji[3] = (j[5] * j[6] - j[3] * j[8]) / det;
    ji[4] = (j[0] * j[8] - j[2] * j[6]) / det;
    ji[5] = (j[2] * j[3] - j[0] * j[5]) / det;
    ji[6] = m2 / det;
    ji[7] = (j[1] * j[6] - j[0] * j[7]) / det;
    ji[8] = (j[0] * j[4] - j[1] * j[3]) / det;
  }
  *det_out = det;
  return det > 0.0;
}

void geometry_tensor(int dim, const double* ji, double det, double* g)
{
  for (int mu = 0; mu < dim; ++mu)
    for (int nu = mu; nu < dim; ++nu)
    {
      double s = 0.0;
      for (int al = 0; al < dim; ++al)
        s = s + ji[mu * dim + al] * ji[nu * dim + al];
      s = s * det;
      g[mu * dim + nu] = g[nu * dim + mu] = s;
    }
}

void check_cells(int dim, const double* v, int64_t nv, const int32_t* cells, int64_t ne)
{
  const int nb = dim + 1;
  for (int64_t e = 0; e < ne; ++e)
  {
    double x[12], j[9], ji[9], det;
    for (int k = 0; k < nb; ++k)
    {
      const int32_t id = cells[e * nb + k];
      if (id < 0 || id >= nv)
        throw std::invalid_argument("cell vertex index " + std::to_string(id) + " out of range");
      for (int c = 0; c < dim; ++c)
        x[k * dim + c] = v[static_cast<int64_t>(id) * dim + c];
    }
    if (!jacobian(dim, x, j, ji, &det))
      throw std::runtime_error("degenerate element: det(J) <= 0 in cell " + std::to_string(e));
  }
}

}  // namespace fbh
