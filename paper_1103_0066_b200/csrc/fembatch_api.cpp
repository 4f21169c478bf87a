// fembatch_api.cpp -- the reference-compatible C++ API (include/fembatch_b200.hpp)
// on top of the C ABI.  Validation order and exception texts follow the
// reference (src/engine.cpp, src/geometry.cpp, src/forms.cpp,
// src/kernel_config.cpp); the integration calls run on the GPU.
#include "../../include/fembatch_b200.hpp"

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <iomanip>
#include <istream>
#include <limits>
#include <ostream>
#include <stdexcept>
#include <string>

#include "../../include/fembatch_b200.h"
#include "fb_host.h"

namespace fembatch {

namespace {

[[noreturn]] void rethrow(const fb_error& e)
{
  switch (e.code)
  {
  case FB_ERR_INVALID_ARGUMENT:
    throw std::invalid_argument(e.message);
  case FB_ERR_OUT_OF_RANGE:
    throw std::out_of_range(e.message);
  default:
    throw std::runtime_error(e.message);
  }
}

void check(int rc, const fb_error& e)
{
  if (rc != FB_OK)
    rethrow(e);
}

int prec_code(Precision p) { return p == Precision::f32 ? FB_F32 : FB_F64; }

fb_kernel_config to_c(const KernelConfig& c)
{
  fb_kernel_config k{};
  k.element_batch_size = c.element_batch_size;
  k.num_concurrent_elements = c.num_concurrent_elements;
  k.interleave_stores = c.interleave_stores ? 1 : 0;
  k.loop_unroll = c.loop_unroll ? 1 : 0;
  k.precision = prec_code(c.precision);
  k.mode = c.mode == Mode::fast ? FB_FAST : FB_STRICT;
  k.store = FB_STORE_AUTO;
  return k;
}

std::vector<int> devices_for(int workers)
{
  if (workers < 1)
    throw std::invalid_argument("worker count must be >= 1");
  const int have = fb_device_count();
  if (have < 1)
    throw std::runtime_error("no CUDA device available");
  std::vector<int> d;
  for (int i = 0; i < std::min(workers, have); ++i)
    d.push_back(i);
  return d;
}

void* data_ptr(ScalarArray& a)
{
  return std::visit([](auto& v) -> void* { return v.data(); }, a);
}
const void* data_ptr(const ScalarArray& a)
{
  return std::visit([](const auto& v) -> const void* { return v.data(); }, a);
}

}  // namespace

// ------------------------------------------------------------ kernel_config
const char* precision_name(Precision p) { return p == Precision::f32 ? "f32" : "f64"; }

Precision precision_from_name(std::string_view name)
{
  if (name == "f32")
    return Precision::f32;
  if (name == "f64")
    return Precision::f64;
  throw std::invalid_argument("unknown precision name: " + std::string(name));
}

std::int64_t scalar_array_size(const ScalarArray& a)
{
  return std::visit([](const auto& v) { return static_cast<std::int64_t>(v.size()); }, a);
}

double scalar_array_at(const ScalarArray& a, std::int64_t i)
{
  return std::visit([i](const auto& v) { return static_cast<double>(v[static_cast<std::size_t>(i)]); }, a);
}

ScalarArray make_scalar_array(Precision p, std::int64_t n)
{
  if (p == Precision::f32)
    return std::vector<float>(static_cast<std::size_t>(n));
  return std::vector<double>(static_cast<std::size_t>(n));
}

void KernelConfig::validate() const
{
  if (element_batch_size < 1)
    throw std::invalid_argument("element_batch_size must be positive");
  if (num_concurrent_elements < 1)
    throw std::invalid_argument("num_concurrent_elements must be positive");
  if (element_batch_size % num_concurrent_elements != 0)
    throw std::invalid_argument("num_concurrent_elements (" + std::to_string(num_concurrent_elements)
                                + ") must divide element_batch_size (" + std::to_string(element_batch_size)
                                + ")");
}

// ---------------------------------------------------------------- reference
ReferenceCell make_reference_cell(int dim)
{
  fbh::check_dim(dim);
  ReferenceCell c;
  c.dim = dim;
  if (dim == 2)
  {
    c.vertices = {0, 0, 1, 0, 0, 1};
    c.volume = 0.5;
  }
  else
  {
    c.vertices = {0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0, 1};
    c.volume = 1.0 / 6.0;
  }
  return c;
}

QuadratureRule make_quadrature(int dim, int degree)
{
  QuadratureRule r;
  r.dim = dim;
  r.degree = degree;
  fbh::quadrature(dim, degree, r.points, r.weights);
  return r;
}

// phi_0 = 1 - sum(xi), phi_{d+1} = xi_d; gradients (-1, ..., -1) and e_d
// (reference include/fembatch/reference.hpp:57-59).
TabulatedBasis tabulate_p1_basis(const ReferenceCell& cell, const QuadratureRule& rule)
{
  if (cell.dim != rule.dim)
    throw std::invalid_argument("cell and rule dimensions differ");
  TabulatedBasis t;
  t.dim = cell.dim;
  t.num_basis_funcs = cell.dim + 1;
  t.num_points = rule.num_points();
  const std::size_t nq = static_cast<std::size_t>(t.num_points);
  t.values.assign((cell.dim + 1) * nq, 0.0);
  t.gradients.assign((cell.dim + 1) * nq * cell.dim, 0.0);
  for (std::size_t q = 0; q < nq; ++q)
  {
    double rest = 1.0;
    for (int d = 0; d < cell.dim; ++d)
    {
      rest -= rule.point(static_cast<int>(q), d);
      t.values[(d + 1) * nq + q] = rule.point(static_cast<int>(q), d);
      t.gradients[q * cell.dim + d] = -1.0;
      t.gradients[((d + 1) * nq + q) * cell.dim + d] = 1.0;
    }
    t.values[q] = rest;
  }
  return t;
}

JetProductTensor integrate_jet_product(const TabulatedBasis& basis, const QuadratureRule& rule,
                                       std::span<const JetFactor> factors)
{
  if (factors.empty())
    throw std::invalid_argument("jet product needs at least one factor");
  if (basis.dim != rule.dim || basis.num_points != rule.num_points())
    throw std::invalid_argument("basis was tabulated for a different rule");
  int slots = 0, values = 0;
  for (const JetFactor& f : factors)
  {
    if (f.slot < 0)
      throw std::invalid_argument("negative basis slot");
    slots = std::max(slots, f.slot + 1);
    values += f.part == JetPart::value ? 1 : 0;  // P1: values degree 1, derivatives degree 0
  }
  for (int sl = 0; sl < slots; ++sl)
    if (std::none_of(factors.begin(), factors.end(), [&](const JetFactor& f) { return f.slot == sl; }))
      throw std::invalid_argument("factor slots must cover 0..S-1");
  if (rule.degree < values)
    throw std::invalid_argument("quadrature degree " + std::to_string(rule.degree)
                                + " insufficient for integrand degree " + std::to_string(values));
  JetProductTensor t;
  t.extents.assign(slots, basis.num_basis_funcs);
  for (const JetFactor& f : factors)
    if (f.part == JetPart::gradient)
      t.extents.push_back(basis.dim);
  std::int64_t n = 1;
  for (int e : t.extents)
    n *= e;
  t.data.assign(static_cast<std::size_t>(n), 0.0);
  std::vector<int> idx(t.extents.size(), 0);  // odometer over the result, last index fastest
  for (std::int64_t flat = 0; flat < n; ++flat)
  {
    double acc = 0.0;
    for (int q = 0; q < rule.num_points(); ++q)
    {
      double prod = 1.0;
      int d = slots;  // next direction index
      for (const JetFactor& f : factors)
        prod *= f.part == JetPart::value ? basis.value(idx[f.slot], q) : basis.gradient(idx[f.slot], q, idx[d++]);
      acc += rule.weights[q] * prod;
    }
    t.data[static_cast<std::size_t>(flat)] = acc;
    for (int k = static_cast<int>(idx.size()) - 1; k >= 0 && ++idx[k] == t.extents[k]; --k)
      idx[k] = 0;
  }
  return t;
}

void dump_analytic_tensor(std::ostream& os, const AnalyticTensor& k)
{
  const FormSpec& sp = k.spec;
  os << "# " << operator_name(sp.op) << " dim=" << sp.dim << " krows=" << sp.krows()
     << " coefficient_blocks=" << sp.num_coefficient_blocks() << "\n";
  char buf[64];
  for (int i = 0; i < sp.krows(); ++i)
    for (int j = 0; j < sp.krows(); ++j)
      for (int c = 0; c < sp.num_coefficient_blocks(); ++c)
      {
        os << "block i=" << i << " j=" << j;
        if (sp.coefficient_arity > 0)
          os << " k=" << c;
        os << "\n";
        for (int mu = 0; mu < sp.dim; ++mu)
        {
          for (int nu = 0; nu < sp.dim; ++nu)
          {
            std::snprintf(buf, sizeof buf, "%s%.17g", nu == 0 ? "" : " ", k.entry(i, j, c, mu, nu));
            os << buf;
          }
          os << "\n";
        }
        os << "\n";
      }
}

// -------------------------------------------------------------------- forms
const char* operator_name(Operator op)
{
  switch (op)
  {
  case Operator::laplacian:
    return "laplacian";
  case Operator::elasticity:
    return "elasticity";
  case Operator::weighted_laplacian:
    return "weighted-laplacian";
  }
  throw std::invalid_argument("unknown operator");
}

Operator operator_from_name(std::string_view name)
{
  if (name == "laplacian")
    return Operator::laplacian;
  if (name == "elasticity")
    return Operator::elasticity;
  if (name == "weighted-laplacian")
    return Operator::weighted_laplacian;
  throw std::invalid_argument("unknown operator name: " + std::string(name));
}

FormSpec make_form_spec(Operator op, int dim)
{
  fbh::check_dim(dim);
  FormSpec s;
  s.op = op;
  s.dim = dim;
  s.num_basis_funcs = dim + 1;
  s.num_components = op == Operator::elasticity ? dim : 1;
  s.coefficient_arity = op == Operator::weighted_laplacian ? 1 : 0;
  s.geometry_arity = 2;
  return s;
}

std::int64_t AnalyticTensor::block_offset(int i, int j, int k) const
{
  return ((i + static_cast<std::int64_t>(j) * spec.krows()) * spec.num_coefficient_blocks() + k) * spec.dim
         * spec.dim;
}

double AnalyticTensor::entry(int i, int j, int k, int mu, int nu) const
{
  return blocks[static_cast<std::size_t>(block_offset(i, j, k) + mu * spec.dim + nu)];
}

AnalyticTensor build_analytic_tensor(Operator op, int dim)
{
  AnalyticTensor k;
  k.spec = make_form_spec(op, dim);
  k.blocks = fbh::build_analytic_tensor(static_cast<int>(op), dim);
  return k;
}
AnalyticTensor build_k_laplacian(int dim) { return build_analytic_tensor(Operator::laplacian, dim); }
AnalyticTensor build_k_elasticity(int dim) { return build_analytic_tensor(Operator::elasticity, dim); }
AnalyticTensor build_k_weighted_laplacian(int dim)
{
  return build_analytic_tensor(Operator::weighted_laplacian, dim);
}

// ----------------------------------------------------------------- geometry
void validate_mesh(const Mesh& mesh)
{
  fbh::check_dim(mesh.dim);
  if (mesh.vertices.size() % mesh.dim != 0)
    throw std::invalid_argument("vertex array length not a multiple of dim");
  if (mesh.cells.size() % (mesh.dim + 1) != 0)
    throw std::invalid_argument("cell array length not a multiple of dim+1");
  fbh::check_cells(mesh.dim, mesh.vertices.data(), mesh.num_vertices(), mesh.cells.data(), mesh.num_elements());
}

Mesh structured_simplicial_mesh(int dim, int n)
{
  std::int64_t nv = 0, ne = 0;
  fbh::structured_mesh_sizes(dim, n, nv, ne);
  Mesh m;
  m.dim = dim;
  m.vertices.resize(static_cast<std::size_t>(nv * dim));
  m.cells.resize(static_cast<std::size_t>(ne * (dim + 1)));
  fbh::structured_mesh(dim, n, m.vertices.data(), m.cells.data());
  return m;
}

Mesh jitter_mesh(const Mesh& mesh, double magnitude, std::uint64_t seed)
{
  Mesh out = mesh;
  fbh::jitter_mesh(out.dim, out.vertices.data(), out.num_vertices(), out.cells.data(), out.num_elements(),
                   magnitude, seed);
  return out;
}

ElementJacobian jacobian_from_vertices(int dim, const double* x)
{
  fbh::check_dim(dim);
  ElementJacobian jac;
  jac.dim = dim;
  if (!fbh::jacobian(dim, x, jac.j.data(), jac.jinv.data(), &jac.det))
    throw std::runtime_error("degenerate element: det(J) <= 0");
  return jac;
}

ElementJacobian element_jacobian(const Mesh& mesh, std::int64_t cell)
{
  if (cell < 0 || cell >= mesh.num_elements())
    throw std::out_of_range("cell index out of range");
  double x[12];
  for (int k = 0; k <= mesh.dim; ++k)
    for (int c = 0; c < mesh.dim; ++c)
      x[k * mesh.dim + c] = mesh.vertex(mesh.cell_vertex(cell, k), c);
  ElementJacobian jac;
  jac.dim = mesh.dim;
  if (!fbh::jacobian(mesh.dim, x, jac.j.data(), jac.jinv.data(), &jac.det))
    throw std::runtime_error("degenerate element: det(J) <= 0 in cell " + std::to_string(cell));
  return jac;
}

GeometryTensor geometry_tensor(const ElementJacobian& jac)
{
  GeometryTensor g;
  g.dim = jac.dim;
  fbh::geometry_tensor(jac.dim, jac.jinv.data(), jac.det, g.g.data());
  return g;
}

std::int64_t packed_geometry_index(int dim, int bs, std::int64_t batch, int e, int mu, int nu)
{
  return (batch * bs + e) * dim * dim + mu * dim + nu;
}

PackedGeometry pack_geometry(const Mesh& mesh, const KernelConfig& config)
{
  fbh::check_dim(mesh.dim);
  config.validate();
  PackedGeometry p;
  p.dim = mesh.dim;
  p.element_batch_size = config.element_batch_size;
  p.num_elements = mesh.num_elements();
  p.num_batches = (p.num_elements + config.element_batch_size - 1) / config.element_batch_size;
  p.precision = config.precision;
  const std::int64_t len = p.num_batches * config.element_batch_size * mesh.dim * mesh.dim;
  p.data = make_scalar_array(config.precision, len);
  if (len == 0)
    return p;
  fb_mesh_view mv{mesh.dim, 0, mesh.num_vertices(), mesh.num_elements(), mesh.vertices.data(), mesh.cells.data()};
  fb_error err{};
  const std::vector<int> dev = devices_for(1);
  check(fb_pack_geometry(&mv, config.element_batch_size, prec_code(config.precision), data_ptr(p.data), len,
                         dev.data(), 1, &err),
        err);
  return p;
}

void write_mesh_text(std::ostream& os, const Mesh& mesh)
{
  os << std::setprecision(std::numeric_limits<double>::max_digits10);
  os << mesh.dim << " " << mesh.num_vertices() << " " << mesh.num_elements() << "\n";
  for (std::int64_t v = 0; v < mesh.num_vertices(); ++v)
  {
    for (int c = 0; c < mesh.dim; ++c)
      os << (c ? " " : "") << mesh.vertex(v, c);
    os << "\n";
  }
  for (std::int64_t e = 0; e < mesh.num_elements(); ++e)
  {
    for (int k = 0; k <= mesh.dim; ++k)
      os << (k ? " " : "") << mesh.cell_vertex(e, k);
    os << "\n";
  }
}

Mesh read_mesh_text(std::istream& is)
{
  Mesh m;
  std::int64_t nv = 0, ne = 0;
  if (!(is >> m.dim >> nv >> ne) || nv < 0 || ne < 0)
    throw std::runtime_error("malformed mesh header");
  fbh::check_dim(m.dim);
  m.vertices.resize(static_cast<std::size_t>(nv * m.dim));
  for (double& x : m.vertices)
    if (!(is >> x))
      throw std::runtime_error("truncated vertex data");
  m.cells.resize(static_cast<std::size_t>(ne * (m.dim + 1)));
  for (std::int32_t& v : m.cells)
    if (!(is >> v))
      throw std::runtime_error("truncated cell data");
  validate_mesh(m);
  return m;
}

// ------------------------------------------------------------------- engine
std::int64_t element_matrix_index(int krows, int bs, int ce, std::int64_t element, int i, int j)
{
  return fb_element_matrix_index(krows, bs, ce, element, i, j);
}

KernelVariant specialize_kernel(const FormSpec& spec, const AnalyticTensor& k, const KernelConfig& config)
{
  config.validate();
  if (!(k.spec == spec))
    throw std::invalid_argument("analytic tensor was built for a different form");
  const fb_kernel_config c = to_c(config);
  fb_error err{};
  fb_variant* v = fb_specialize(static_cast<int>(spec.op), spec.dim, k.blocks.data(),
                                static_cast<std::int64_t>(k.blocks.size()), &c, &err);
  if (!v)
    rethrow(err);
  KernelVariant out;
  out.spec = spec;
  out.config = config;
  out.device = std::shared_ptr<fb_variant>(v, fb_variant_free);
  out.description = fb_variant_description(v);
  out.k = make_scalar_array(config.precision, static_cast<std::int64_t>(k.blocks.size()));
  std::visit(
      [&](auto& dst)
      {
        using S = typename std::decay_t<decltype(dst)>::value_type;
        for (std::size_t t = 0; t < k.blocks.size(); ++t)
          dst[t] = static_cast<S>(k.blocks[t]);
      },
      out.k);
  return out;
}

namespace {

ElementMatrixStore empty_store(const KernelVariant& v, std::int64_t num_batches, std::int64_t ne)
{
  ElementMatrixStore s;
  s.dim = v.spec.dim;
  s.krows = v.spec.krows();
  s.element_batch_size = v.config.element_batch_size;
  s.num_concurrent_elements = v.config.num_concurrent_elements;
  s.num_batches = num_batches;
  s.num_elements = ne;
  s.precision = v.config.precision;
  s.data = make_scalar_array(v.config.precision,
                             num_batches * v.config.element_batch_size * s.krows * s.krows);
  return s;
}

const double* coefficient_ptr(const KernelVariant& v, const CoefficientField* w, std::int64_t ne)
{
  if (v.spec.coefficient_arity == 1)
  {
    if (w == nullptr)
      throw std::invalid_argument("form requires a coefficient field");
    if (w->num_basis_funcs != v.spec.num_basis_funcs)
      throw std::invalid_argument("coefficient field has wrong block size");
    if (static_cast<std::int64_t>(w->values.size()) < ne * v.spec.num_basis_funcs)
      throw std::invalid_argument("coefficient field is shorter than the mesh");
    if (ne == 0)
      throw std::invalid_argument("cannot integrate a coefficient form over zero elements");
    return w->values.data();
  }
  if (w != nullptr)
    throw std::invalid_argument("form takes no coefficient field");
  return nullptr;
}

}  // namespace

ElementMatrixStore integrate_batches(const KernelVariant& v, const PackedGeometry& geom,
                                     const CoefficientField* coefficients, int workers)
{
  v.config.validate();
  if (geom.dim != v.spec.dim)
    throw std::invalid_argument("geometry dimension does not match form");
  if (geom.element_batch_size != v.config.element_batch_size)
    throw std::invalid_argument("geometry was packed for a different batch size");
  if (geom.precision != v.config.precision)
    throw std::invalid_argument("geometry was packed in a different precision");
  if (workers < 1)
    throw std::invalid_argument("worker count must be >= 1");
  const double* w = coefficient_ptr(v, coefficients, geom.num_elements);
  if (!v.device)
    throw std::invalid_argument("kernel variant was not specialized for the GPU");
  ElementMatrixStore s = empty_store(v, geom.num_batches, geom.num_elements);
  const std::int64_t len = scalar_array_size(s.data);
  if (len == 0)
    return s;
  const std::vector<int> dev = devices_for(workers);
  fb_error err{};
  check(fb_integrate_packed(v.device.get(), geom.dim, data_ptr(geom.data), geom.num_batches, geom.num_elements,
                            w, data_ptr(s.data), len, dev.data(), static_cast<int>(dev.size()), &err),
        err);
  return s;
}

ElementMatrixStore integrate_mesh(const KernelVariant& v, const Mesh& mesh, const CoefficientField* coefficients,
                                  int workers)
{
  v.config.validate();
  if (mesh.dim != v.spec.dim)
    throw std::invalid_argument("geometry dimension does not match form");
  if (workers < 1)
    throw std::invalid_argument("worker count must be >= 1");
  const double* w = coefficient_ptr(v, coefficients, mesh.num_elements());
  if (!v.device)
    throw std::invalid_argument("kernel variant was not specialized for the GPU");
  const std::int64_t ne = mesh.num_elements();
  const int bs = v.config.element_batch_size;
  ElementMatrixStore s = empty_store(v, (ne + bs - 1) / bs, ne);
  const std::int64_t len = scalar_array_size(s.data);
  if (len == 0)
    return s;
  const std::vector<int> dev = devices_for(workers);
  fb_mesh_view mv{mesh.dim, 0, mesh.num_vertices(), ne, mesh.vertices.data(), mesh.cells.data()};
  fb_error err{};
  check(fb_integrate_mesh(v.device.get(), &mv, w, data_ptr(s.data), len, dev.data(), static_cast<int>(dev.size()),
                          &err),
        err);
  return s;
}

std::int64_t flop_count(const FormSpec& spec, const KernelConfig&, std::int64_t ne)
{
  return fb_flop_count(static_cast<int>(spec.op), spec.dim, ne);
}

std::vector<double> unpack_element_matrix(const ElementMatrixStore& store, const KernelConfig& config,
                                          const FormSpec& spec, std::int64_t element)
{
  if (spec.krows() != store.krows || spec.dim != store.dim)
    throw std::invalid_argument("store does not match form");
  if (config.element_batch_size != store.element_batch_size
      || config.num_concurrent_elements != store.num_concurrent_elements)
    throw std::invalid_argument("store does not match kernel config");
  if (element < 0 || element >= store.num_elements)
    throw std::out_of_range("element index out of range");
  const int kr = store.krows;
  std::vector<double> m(static_cast<std::size_t>(kr) * kr);
  for (int i = 0; i < kr; ++i)
    for (int j = 0; j < kr; ++j)
      m[static_cast<std::size_t>(i) * kr + j] = scalar_array_at(
          store.data, element_matrix_index(kr, store.element_batch_size, store.num_concurrent_elements, element,
                                           i, j));
  return m;
}

// FBEMAT01 store format (reference src/engine.cpp:413-508): magic, dim, krows,
// bs, ce (u32), num_elements (u64), precision (u32: 0 f32, 1 f64), scalars;
// little-endian.
namespace {
constexpr char kMagic[8] = {'F', 'B', 'E', 'M', 'A', 'T', '0', '1'};
template <class T>
void put(std::ostream& os, T v)
{
  os.write(reinterpret_cast<const char*>(&v), sizeof v);
}
template <class T>
T get(std::istream& is)
{
  T v{};
  is.read(reinterpret_cast<char*>(&v), sizeof v);
  return v;
}
}  // namespace

void write_store(std::ostream& os, const ElementMatrixStore& s)
{
  os.write(kMagic, 8);
  put<std::uint32_t>(os, static_cast<std::uint32_t>(s.dim));
  put<std::uint32_t>(os, static_cast<std::uint32_t>(s.krows));
  put<std::uint32_t>(os, static_cast<std::uint32_t>(s.element_batch_size));
  put<std::uint32_t>(os, static_cast<std::uint32_t>(s.num_concurrent_elements));
  put<std::uint64_t>(os, static_cast<std::uint64_t>(s.num_elements));
  put<std::uint32_t>(os, s.precision == Precision::f32 ? 0u : 1u);
  const std::int64_t n = scalar_array_size(s.data);
  os.write(static_cast<const char*>(data_ptr(s.data)),
           static_cast<std::streamsize>(n * (s.precision == Precision::f32 ? 4 : 8)));
  if (!os)
    throw std::runtime_error("failed to write element-matrix store");
}

ElementMatrixStore read_store(std::istream& is)
{
  char magic[8] = {};
  is.read(magic, 8);
  if (!is || std::memcmp(magic, kMagic, 8) != 0)
    throw std::runtime_error("not an element-matrix store file");
  ElementMatrixStore s;
  s.dim = static_cast<int>(get<std::uint32_t>(is));
  s.krows = static_cast<int>(get<std::uint32_t>(is));
  s.element_batch_size = static_cast<int>(get<std::uint32_t>(is));
  s.num_concurrent_elements = static_cast<int>(get<std::uint32_t>(is));
  s.num_elements = static_cast<std::int64_t>(get<std::uint64_t>(is));
  const std::uint32_t pc = get<std::uint32_t>(is);
  if (!is)
    throw std::runtime_error("truncated element-matrix store header");
  if (s.dim != 2 && s.dim != 3)
    throw std::runtime_error("store header: bad dimension");
  if (s.krows <= 0 || s.element_batch_size <= 0 || s.num_concurrent_elements <= 0 || s.num_elements < 0
      || s.element_batch_size % s.num_concurrent_elements != 0)
    throw std::runtime_error("store header: bad batch shape");
  if (pc > 1)
    throw std::runtime_error("store header: bad precision code");
  s.precision = pc == 0 ? Precision::f32 : Precision::f64;
  s.num_batches = (s.num_elements + s.element_batch_size - 1) / s.element_batch_size;
  s.data = make_scalar_array(s.precision,
                             s.num_batches * static_cast<std::int64_t>(s.krows) * s.krows * s.element_batch_size);
  is.read(static_cast<char*>(data_ptr(s.data)),
          static_cast<std::streamsize>(scalar_array_size(s.data) * (pc == 0 ? 4 : 8)));
  if (!is)
    throw std::runtime_error("truncated element-matrix store data");
  return s;
}

// ---- global assembly ------------------------------------------------------
AssemblyPlan make_assembly_plan(Operator op, const Mesh& mesh)
{
  fb_error err{};
  fb_assembly* a = fb_assembly_create(static_cast<int>(op), mesh.dim, mesh.cells.data(), mesh.num_elements(),
                                      mesh.num_vertices(), &err);
  if (!a)
    check(err.code ? err.code : FB_ERR_INVALID_ARGUMENT, err);
  AssemblyPlan p;
  p.op = op;
  p.dim = mesh.dim;
  p.device = std::shared_ptr<fb_assembly>(a, fb_assembly_free);
  p.rows = fb_assembly_rows(a);
  p.nnz = fb_assembly_nnz(a);
  return p;
}

CsrMatrix assemble_global(const KernelVariant& v, const AssemblyPlan& plan, const ElementMatrixStore& store,
                          bool symmetric, int device, bool block_diagonal)
{
  if (!v.device || !plan.device)
    throw std::invalid_argument("variant or assembly plan was not created for the GPU");
  if (store.precision != v.config.precision || store.dim != plan.dim)
    throw std::invalid_argument("store does not match variant / plan");
  CsrMatrix m;
  m.rows = plan.rows;
  m.precision = store.precision;
  m.row_ptr.resize(plan.rows + 1);
  m.col_idx.resize(plan.nnz);
  fb_error err{};
  check(fb_assembly_pattern(plan.device.get(), m.row_ptr.data(), plan.rows + 1, m.col_idx.data(), plan.nnz, &err),
        err);
  m.values = make_scalar_array(store.precision, plan.nnz);
  check(fb_assemble(plan.device.get(), v.device.get(), data_ptr(store.data),
                    scalar_array_size(store.data), data_ptr(m.values), plan.nnz,
                    (symmetric ? FB_ASSEMBLE_SYMMETRIC : 0) | (block_diagonal ? FB_ASSEMBLE_BLOCK_DIAGONAL : 0),
                    device, &err),
        err);
  return m;
}

CsrMatrix assemble_global(const KernelVariant& v, const AssemblyPlan& plan, const PackedGeometry& geometry,
                          const std::vector<double>& coefficients, int device)
{
  if (!v.device || !plan.device)
    throw std::invalid_argument("variant or assembly plan was not created for the GPU");
  if (geometry.precision != v.config.precision || geometry.dim != plan.dim)
    throw std::invalid_argument("packed geometry does not match variant / plan");
  CsrMatrix m;
  m.rows = plan.rows;
  m.precision = geometry.precision;
  m.row_ptr.resize(plan.rows + 1);
  m.col_idx.resize(plan.nnz);
  fb_error err{};
  check(fb_assembly_pattern(plan.device.get(), m.row_ptr.data(), plan.rows + 1, m.col_idx.data(), plan.nnz, &err),
        err);
  m.values = make_scalar_array(geometry.precision, plan.nnz);
  check(fb_assemble_packed(plan.device.get(), v.device.get(), data_ptr(geometry.data),
                           scalar_array_size(geometry.data), coefficients.empty() ? nullptr : coefficients.data(),
                           static_cast<std::int64_t>(coefficients.size()), data_ptr(m.values), plan.nnz, device,
                           &err),
        err);
  return m;
}

}  // namespace fembatch
