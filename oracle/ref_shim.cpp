// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" wrappers that drive the UNMODIFIED reference fembatch library
// (compiled from /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libfembatch_ref.so).  Used (a) to pin the C restatement in
// oracle/fb_oracle.c, (b) to generate tests/golden/, and (c) as the CPU
// baseline / `bench.py --impl reference` arm.  Nothing here is part of the
// product library.
#include <chrono>
#include <fstream>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "fembatch/bench.hpp"
#include "fembatch/engine.hpp"
#include "fembatch/forms.hpp"
#include "fembatch/geometry.hpp"
#include "fembatch/oracle.hpp"

using namespace fembatch;

namespace {

thread_local std::string g_last_error;

int fail(const std::exception& e)
{
  g_last_error = e.what();
  return -1;
}

Mesh mesh_from(int dim, const double* v, std::int64_t nv, const std::int32_t* c,
               std::int64_t ne)
{
  Mesh m;
  m.dim = dim;
  m.vertices.assign(v, v + nv * dim);
  m.cells.assign(c, c + ne * (dim + 1));
  return m;
}

KernelConfig config_from(int bs, int ce, int is, int ur, int precision)
{
  KernelConfig k;
  k.element_batch_size = bs;
  k.num_concurrent_elements = ce;
  k.interleave_stores = is != 0;
  k.loop_unroll = ur != 0;
  k.precision = precision == 0 ? Precision::f32 : Precision::f64;
  return k;
}

void copy_store(const ElementMatrixStore& s, void* out)
{
  std::visit(
      [&](const auto& d)
      {
        std::memcpy(out, d.data(), d.size() * sizeof(d[0]));
      },
      s.data);
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_last_error.c_str(); }

int ref_mesh_sizes(int dim, int n, std::int64_t* nv, std::int64_t* ne)
{
  try
  {
    const std::int64_t m = n + 1;
    *nv = dim == 2 ? m * m : m * m * m;
    *ne = dim == 2 ? 2LL * n * n : 6LL * n * n * n;
    return 0;
  }
  catch (const std::exception& e)
  {
    return fail(e);
  }
}

int ref_make_mesh(int dim, int n, double jitter, std::uint64_t seed,
                  double* vertices, std::int32_t* cells)
{
  try
  {
    Mesh m = structured_simplicial_mesh(dim, n);
    if (jitter > 0.0)
      m = jitter_mesh(m, jitter, seed);
    std::memcpy(vertices, m.vertices.data(), m.vertices.size() * sizeof(double));
    std::memcpy(cells, m.cells.data(), m.cells.size() * sizeof(std::int32_t));
    return 0;
  }
  catch (const std::exception& e)
  {
    return fail(e);
  }
}

std::int64_t ref_k_len(int op, int dim)
{
  const FormSpec s = make_form_spec(static_cast<Operator>(op), dim);
  return static_cast<std::int64_t>(s.krows()) * s.krows()
         * s.num_coefficient_blocks() * dim * dim;
}

int ref_build_k(int op, int dim, double* out)
{
  try
  {
    const AnalyticTensor k = build_analytic_tensor(static_cast<Operator>(op), dim);
    std::memcpy(out, k.blocks.data(), k.blocks.size() * sizeof(double));
    return 0;
  }
  catch (const std::exception& e)
  {
    return fail(e);
  }
}

int ref_jacobian(int dim, const double* coords, double* j, double* jinv,
                 double* det, double* g)
{
  try
  {
    const ElementJacobian jac = jacobian_from_vertices(dim, coords);
    const GeometryTensor gt = geometry_tensor(jac);
    for (int t = 0; t < dim * dim; ++t)
    {
      j[t] = jac.j[t];
      jinv[t] = jac.jinv[t];
      g[t] = gt.g[t];
    }
    *det = jac.det;
    return 0;
  }
  catch (const std::exception& e)
  {
    return fail(e);
  }
}

int ref_pack_geometry(int dim, const double* v, std::int64_t nv,
                      const std::int32_t* c, std::int64_t ne, int bs,
                      int precision, void* out)
{
  try
  {
    const Mesh m = mesh_from(dim, v, nv, c, ne);
    const PackedGeometry g = pack_geometry(m, config_from(bs, 1, 0, 0, precision));
    std::visit(
        [&](const auto& d) { std::memcpy(out, d.data(), d.size() * sizeof(d[0])); },
        g.data);
    return 0;
  }
  catch (const std::exception& e)
  {
    return fail(e);
  }
}

// pack_geometry + integrate_batches (the library composition every reference
// caller uses, tests/test_engine.cpp:28-38).  out holds num_batches*bs*nk
// scalars of the engine precision.
int ref_integrate_mesh(int op, int dim, const double* v, std::int64_t nv,
                       const std::int32_t* c, std::int64_t ne, int bs, int ce,
                       int is, int ur, int precision, int workers,
                       const double* coeffs, void* out)
{
  try
  {
    const Mesh m = mesh_from(dim, v, nv, c, ne);
    const FormSpec spec = make_form_spec(static_cast<Operator>(op), dim);
    const AnalyticTensor k = build_analytic_tensor(spec.op, dim);
    const KernelConfig cfg = config_from(bs, ce, is, ur, precision);
    const KernelVariant var = specialize_kernel(spec, k, cfg);
    const PackedGeometry g = pack_geometry(m, cfg);
    CoefficientField w;
    const CoefficientField* wp = nullptr;
    if (spec.coefficient_arity == 1)
    {
      w.num_basis_funcs = spec.num_basis_funcs;
      w.values.assign(coeffs, coeffs + ne * spec.num_basis_funcs);
      wp = &w;
    }
    copy_store(integrate_batches(var, g, wp, workers), out);
    return 0;
  }
  catch (const std::exception& e)
  {
    return fail(e);
  }
}

// The reference's own FBEMAT01 store file (src/engine.cpp:413-508) and text
// mesh file (src/geometry.cpp:353-395) for a structured (jittered) mesh --
// golden files for the F4 format rows.
int ref_write_files(int op, int dim, int n, double jitter, std::uint64_t seed, int bs, int ce, int precision,
                    const char* store_path, const char* mesh_path)
{
  try
  {
    Mesh m = structured_simplicial_mesh(dim, n);
    if (jitter > 0.0)
      m = jitter_mesh(m, jitter, seed);
    const FormSpec spec = make_form_spec(static_cast<Operator>(op), dim);
    const KernelConfig cfg = config_from(bs, ce, 1, 0, precision);
    const KernelVariant var = specialize_kernel(spec, build_analytic_tensor(spec.op, dim), cfg);
    const ElementMatrixStore store = integrate_batches(var, pack_geometry(m, cfg));
    std::ofstream fs(store_path, std::ios::binary);
    write_store(fs, store);
    std::ofstream fm(mesh_path);
    write_mesh_text(fm, m);
    return fs.good() && fm.good() ? 0 : -1;
  }
  catch (const std::exception& e)
  {
    return fail(e);
  }
}

// integrate_batches on caller-provided packed G (slot-major, engine
// precision) -- the synthetic-G path of tests/test_engine.cpp:337-378.
int ref_integrate_packed(int op, int dim, const void* gdata,
                         std::int64_t num_batches, std::int64_t ne, int bs,
                         int ce, int precision, const double* coeffs, void* out)
{
  try
  {
    const FormSpec spec = make_form_spec(static_cast<Operator>(op), dim);
    const AnalyticTensor k = build_analytic_tensor(spec.op, dim);
    const KernelConfig cfg = config_from(bs, ce, 1, 0, precision);
    const KernelVariant var = specialize_kernel(spec, k, cfg);
    PackedGeometry g;
    g.dim = dim;
    g.element_batch_size = bs;
    g.num_batches = num_batches;
    g.num_elements = ne;
    g.precision = cfg.precision;
    const std::int64_t len = num_batches * bs * dim * dim;
    g.data = make_scalar_array(cfg.precision, len);
    std::visit(
        [&](auto& d) { std::memcpy(d.data(), gdata, d.size() * sizeof(d[0])); },
        g.data);
    CoefficientField w;
    const CoefficientField* wp = nullptr;
    if (spec.coefficient_arity == 1)
    {
      w.num_basis_funcs = spec.num_basis_funcs;
      w.values.assign(coeffs, coeffs + ne * spec.num_basis_funcs);
      wp = &w;
    }
    copy_store(integrate_batches(var, g, wp, 1), out);
    return 0;
  }
  catch (const std::exception& e)
  {
    return fail(e);
  }
}

int ref_direct(int op, int dim, const double* coords, const double* coeffs,
               double* out)
{
  try
  {
    const FormSpec spec = make_form_spec(static_cast<Operator>(op), dim);
    std::span<const double> w;
    if (spec.coefficient_arity == 1)
      w = std::span<const double>(coeffs, spec.num_basis_funcs);
    const std::vector<double> m = assemble_element_direct(
        spec, std::span<const double>(coords, (dim + 1) * dim), w);
    std::memcpy(out, m.data(), m.size() * sizeof(double));
    return 0;
  }
  catch (const std::exception& e)
  {
    return fail(e);
  }
}

int ref_default_coefficients(int dim, const double* v, std::int64_t nv,
                             const std::int32_t* c, std::int64_t ne, double* out)
{
  try
  {
    const CoefficientField f = default_coefficient_field(mesh_from(dim, v, nv, c, ne));
    std::memcpy(out, f.values.data(), f.values.size() * sizeof(double));
    return 0;
  }
  catch (const std::exception& e)
  {
    return fail(e);
  }
}

std::int64_t ref_flop_count(int op, int dim, std::int64_t ne)
{
  return flop_count(make_form_spec(static_cast<Operator>(op), dim), KernelConfig{}, ne);
}

std::int64_t ref_element_matrix_index(int krows, int bs, int ce,
                                      std::int64_t e, int i, int j)
{
  return element_matrix_index(krows, bs, ce, e, i, j);
}

// The reference's own timed path (bench.cpp:150-164 semantics): min and mean
// steady_clock seconds over `reps` of [pack_geometry if include_packing] +
// integrate_batches, with a prepared variant.  Returns 0 on success.
int ref_time_integrate(int op, int dim, const double* v, std::int64_t nv,
                       const std::int32_t* c, std::int64_t ne, int bs, int ce,
                       int is, int ur, int precision, int workers, int reps,
                       int include_packing, const double* coeffs,
                       double* seconds_min, double* seconds_mean)
{
  try
  {
    const Mesh m = mesh_from(dim, v, nv, c, ne);
    const FormSpec spec = make_form_spec(static_cast<Operator>(op), dim);
    const AnalyticTensor k = build_analytic_tensor(spec.op, dim);
    const KernelConfig cfg = config_from(bs, ce, is, ur, precision);
    const KernelVariant var = specialize_kernel(spec, k, cfg);
    CoefficientField w;
    const CoefficientField* wp = nullptr;
    if (spec.coefficient_arity == 1)
    {
      w.num_basis_funcs = spec.num_basis_funcs;
      w.values.assign(coeffs, coeffs + ne * spec.num_basis_funcs);
      wp = &w;
    }
    PackedGeometry g;
    if (!include_packing)
      g = pack_geometry(m, cfg);
    double mn = 0.0, sum = 0.0;
    for (int r = 0; r < reps; ++r)
    {
      const auto t0 = std::chrono::steady_clock::now();
      if (include_packing)
        g = pack_geometry(m, cfg);
      ElementMatrixStore s = integrate_batches(var, g, wp, workers);
      const auto t1 = std::chrono::steady_clock::now();
      const double sec = std::chrono::duration<double>(t1 - t0).count();
      mn = r == 0 ? sec : std::min(mn, sec);
      sum += sec;
    }
    *seconds_min = mn;
    *seconds_mean = sum / reps;
    return 0;
  }
  catch (const std::exception& e)
  {
    return fail(e);
  }
}

}  // extern "C"
