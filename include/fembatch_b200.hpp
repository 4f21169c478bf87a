// fembatch_b200.hpp -- C++ host layer of the B200 engine.
//
// Source-compatible with the reference library's public API
// (/root/reference/proj/include/fembatch/*.hpp): same namespace, type names,
// fields, function signatures and exception types/texts, so a caller of the
// reference recompiles against this header and links libfembatch_b200.so.
// The integration entry points run on B200s through the C ABI in
// fembatch_b200.h; K construction and mesh synthesis stay host precompute.
//
// GPU meaning of the reference knobs:
//   KernelConfig axes   value-neutral, as on the CPU (store length/padding,
//                       validation, variant name); `mode` picks strict
//                       (bitwise reference) or fast (FMA) arithmetic.
//   workers             number of GPUs the element range is sharded over
//                       (contiguous tile-aligned slices, no collectives);
//                       clamped to the devices present.
#pragma once

#include <array>
#include <cstdint>
#include <iosfwd>
#include <memory>
#include <span>
#include <string>
#include <string_view>
#include <variant>
#include <vector>

struct fb_variant;
struct fb_assembly;

namespace fembatch {

// ---- kernel_config (reference include/fembatch/kernel_config.hpp) --------
enum class Precision { f32, f64 };
const char* precision_name(Precision p);
Precision precision_from_name(std::string_view name);

using ScalarArray = std::variant<std::vector<float>, std::vector<double>>;
std::int64_t scalar_array_size(const ScalarArray& a);
double scalar_array_at(const ScalarArray& a, std::int64_t index);
ScalarArray make_scalar_array(Precision p, std::int64_t size);

enum class Mode { strict, fast };  // GPU extension

struct KernelConfig {
  int element_batch_size = 128;
  int num_concurrent_elements = 1;
  bool interleave_stores = false;
  bool loop_unroll = false;
  Precision precision = Precision::f64;
  Mode mode = Mode::strict;  // GPU extension: strict = bitwise reference arithmetic

  int serial_batch_size() const { return element_batch_size / num_concurrent_elements; }
  void validate() const;  // throws std::invalid_argument
};

// ---- reference cell / quadrature (reference include/fembatch/reference.hpp)
struct ReferenceCell {
  int dim = 0;
  std::vector<double> vertices;
  double volume = 0.0;
};
struct QuadratureRule {
  int dim = 0;
  int degree = 0;
  std::vector<double> points;
  std::vector<double> weights;
  int num_points() const { return static_cast<int>(weights.size()); }
  double point(int q, int c) const { return points[static_cast<std::size_t>(q) * dim + c]; }
};
// P1 hat functions at the points of a rule: values [function][point],
// reference gradients [function][point][direction] (constant per function).
struct TabulatedBasis {
  int dim = 0;
  int num_basis_funcs = 0;
  int num_points = 0;
  std::vector<double> values;
  std::vector<double> gradients;
  double value(int f, int q) const { return values[static_cast<std::size_t>(f) * num_points + q]; }
  double gradient(int f, int q, int d) const
  {
    return gradients[(static_cast<std::size_t>(f) * num_points + q) * dim + d];
  }
};
ReferenceCell make_reference_cell(int dim);
QuadratureRule make_quadrature(int dim, int degree);
TabulatedBasis tabulate_p1_basis(const ReferenceCell& cell, const QuadratureRule& rule);

// ---- forms (reference include/fembatch/forms.hpp) -------------------------
enum class Operator { laplacian, elasticity, weighted_laplacian };
const char* operator_name(Operator op);
Operator operator_from_name(std::string_view name);

struct FormSpec {
  Operator op = Operator::laplacian;
  int dim = 0;
  int num_components = 1;
  int num_basis_funcs = 0;
  int coefficient_arity = 0;
  int geometry_arity = 2;
  int krows() const { return num_basis_funcs * num_components; }
  int num_coefficient_blocks() const { return coefficient_arity == 0 ? 1 : num_basis_funcs; }
  friend bool operator==(const FormSpec&, const FormSpec&) = default;
};
FormSpec make_form_spec(Operator op, int dim);

struct AnalyticTensor {
  FormSpec spec;
  std::vector<double> blocks;  // ((i + j*krows)*ncoef + k)*dim^2 + mu*dim + nu
  std::int64_t block_offset(int i, int j, int k = 0) const;
  double entry(int i, int j, int k, int mu, int nu) const;
};
AnalyticTensor build_k_laplacian(int dim);
AnalyticTensor build_k_elasticity(int dim);
AnalyticTensor build_k_weighted_laplacian(int dim);
AnalyticTensor build_analytic_tensor(Operator op, int dim);

// Exact reference-cell quadrature of a product of P1 basis values and
// first derivatives (the building block of K).  Result: one basis index per
// slot (slot order), then one direction index per gradient factor (factor
// order), row-major.
enum class JetPart { value, gradient };
struct JetFactor {
  int slot = 0;
  JetPart part = JetPart::value;
};
struct JetProductTensor {
  std::vector<int> extents;
  std::vector<double> data;
};
JetProductTensor integrate_jet_product(const TabulatedBasis& basis, const QuadratureRule& rule,
                                       std::span<const JetFactor> factors);
// Plain-text dump of K: "# <op> dim=.. krows=.. coefficient_blocks=.." and
// one "block i=.. j=..[ k=..]" stanza per block, rows of 17 significant digits.
void dump_analytic_tensor(std::ostream& os, const AnalyticTensor& k);

// ---- geometry (reference include/fembatch/geometry.hpp) -------------------
struct Mesh {
  int dim = 0;
  std::vector<double> vertices;
  std::vector<std::int32_t> cells;
  std::int64_t num_vertices() const { return dim == 0 ? 0 : static_cast<std::int64_t>(vertices.size()) / dim; }
  std::int64_t num_elements() const
  {
    return dim == 0 ? 0 : static_cast<std::int64_t>(cells.size()) / (dim + 1);
  }
  double vertex(std::int64_t v, int c) const { return vertices[static_cast<std::size_t>(v) * dim + c]; }
  std::int32_t cell_vertex(std::int64_t e, int k) const
  {
    return cells[static_cast<std::size_t>(e) * (dim + 1) + k];
  }
};
void validate_mesh(const Mesh& mesh);
Mesh structured_simplicial_mesh(int dim, int n);
Mesh jitter_mesh(const Mesh& mesh, double magnitude, std::uint64_t seed);

struct ElementJacobian {
  int dim = 0;
  std::array<double, 9> j{};
  std::array<double, 9> jinv{};
  double det = 0.0;
};
ElementJacobian jacobian_from_vertices(int dim, const double* vertex_coords);
ElementJacobian element_jacobian(const Mesh& mesh, std::int64_t cell);

struct GeometryTensor {
  int dim = 0;
  std::array<double, 9> g{};
  double entry(int mu, int nu) const { return g[mu * dim + nu]; }
};
GeometryTensor geometry_tensor(const ElementJacobian& jac);

struct PackedGeometry {
  int dim = 0;
  int element_batch_size = 0;
  std::int64_t num_batches = 0;
  std::int64_t num_elements = 0;
  Precision precision = Precision::f64;
  ScalarArray data;
};
std::int64_t packed_geometry_index(int dim, int element_batch_size, std::int64_t batch,
                                   int element_in_batch, int mu, int nu);
PackedGeometry pack_geometry(const Mesh& mesh, const KernelConfig& config);  // runs on GPU
void write_mesh_text(std::ostream& os, const Mesh& mesh);
Mesh read_mesh_text(std::istream& is);

// ---- engine (reference include/fembatch/engine.hpp) -----------------------
inline constexpr int work_group_bound = 1024;

struct KernelVariant {
  FormSpec spec;
  KernelConfig config;
  ScalarArray k;
  std::string description;
  std::shared_ptr<fb_variant> device;  // GPU extension: validated device variant
};

struct ElementMatrixStore {
  int dim = 0;
  int krows = 0;
  int element_batch_size = 0;
  int num_concurrent_elements = 0;
  std::int64_t num_batches = 0;
  std::int64_t num_elements = 0;
  Precision precision = Precision::f64;
  ScalarArray data;
};

std::int64_t element_matrix_index(int krows, int element_batch_size, int num_concurrent_elements,
                                  std::int64_t element, int i, int j);

struct CoefficientField {
  int num_basis_funcs = 0;
  std::vector<double> values;
};

KernelVariant specialize_kernel(const FormSpec& spec, const AnalyticTensor& k, const KernelConfig& config);
ElementMatrixStore integrate_batches(const KernelVariant& variant, const PackedGeometry& geom,
                                     const CoefficientField* coefficients = nullptr, int workers = 1);
// Fused mesh -> matrices (GPU extension; equals pack_geometry + integrate_batches
// bitwise in strict mode, without ever materialising G).
ElementMatrixStore integrate_mesh(const KernelVariant& variant, const Mesh& mesh,
                                  const CoefficientField* coefficients = nullptr, int workers = 1);
std::int64_t flop_count(const FormSpec& spec, const KernelConfig& config, std::int64_t num_elements);
std::vector<double> unpack_element_matrix(const ElementMatrixStore& store, const KernelConfig& config,
                                          const FormSpec& spec, std::int64_t element);
void write_store(std::ostream& os, const ElementMatrixStore& store);
ElementMatrixStore read_store(std::istream& is);

// ---- global assembly (GPU extension; SURVEY 8f row F3 -- the reference's
// declared non-goal).  dof(v, c) = v*nc + c, nc = dim for
// elasticity else 1; values = the serial element-order sum, bitwise.
struct CsrMatrix {
  std::int64_t rows = 0;
  std::vector<std::int64_t> row_ptr;
  std::vector<std::int32_t> col_idx;
  Precision precision = Precision::f64;
  ScalarArray values;
};

struct AssemblyPlan {
  Operator op = Operator::laplacian;
  int dim = 0;
  std::int64_t rows = 0, nnz = 0;
  std::shared_ptr<fb_assembly> device;  // pattern + incidence lists (host built, uploaded per device)
};

AssemblyPlan make_assembly_plan(Operator op, const Mesh& mesh);
// `store` must hold the element matrices of the plan's mesh (e.g. from
// integrate_mesh); `symmetric` = every element matrix is bitwise symmetric
// (true for integrate_mesh output of the reference forms), read as columns.
// `block_diagonal` (elasticity) = every element matrix is zero off the
// component diagonal with equal diagonal blocks (true for integrate_mesh
// output of a P1-sparse variant): only block (0,0) of the store is read.
CsrMatrix assemble_global(const KernelVariant& variant, const AssemblyPlan& plan, const ElementMatrixStore& store,
                          bool symmetric = false, int device = 0, bool block_diagonal = false);
// The same operator straight from packed geometry (fb_assemble_packed): the
// element matrices are recomputed per incidence and never stored; bitwise
// assemble_global(integrate_batches(geometry)).  Needs a P1-pattern K.
CsrMatrix assemble_global(const KernelVariant& variant, const AssemblyPlan& plan, const PackedGeometry& geometry,
                          const std::vector<double>& coefficients = {}, int device = 0);

// ---- benchmark records (reference include/fembatch/bench.hpp) ------------
// The record and its CSV / JSON forms, field for field
// the reference's, and the store checksum (row A16).  The benchmark RUNNER
// (run_benchmark, sweep) and the verification module are reference tooling
// outside the hot path: they live in the separate compatibility library
// (include/fembatch_compat.hpp, compat/libfembatch_compat.so).
struct BenchRecord {
  std::string op;
  int dim = 0;
  std::int64_t num_elements = 0;
  int batch_size = 0;
  int concurrent = 0;
  bool interleave = false;
  bool unroll = false;
  std::string precision;
  int workers = 0;
  int reps = 0;
  double seconds_min = 0.0;
  double seconds_mean = 0.0;
  double gflops = 0.0;
  double checksum = 0.0;
  std::string status;
  friend bool operator==(const BenchRecord&, const BenchRecord&) = default;
};
CoefficientField default_coefficient_field(const Mesh& mesh);  // w = 1 + x0 at cell vertices
double store_checksum(const ElementMatrixStore& store);        // real entries, element order, in double
double default_tolerance(Precision p);                         // 1e-12 f64, 5e-5 f32
extern const char* const csv_header;
void write_csv(std::ostream& os, const std::vector<BenchRecord>& records);
std::vector<BenchRecord> read_csv(std::istream& is);
void write_json(std::ostream& os, const std::vector<BenchRecord>& records);

}  // namespace fembatch
