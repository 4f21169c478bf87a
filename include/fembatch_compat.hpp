// fembatch_compat.hpp -- reference tooling on top of the B200 engine, kept
// OUT of the product library (libfembatch_b200.so): the benchmark runner and
// variant sweep (reference include/fembatch/bench.hpp, src/bench.cpp) and the
// verification module (include/fembatch/oracle.hpp, src/oracle.cpp).  Built
// as compat/libfembatch_compat.so (compat/Makefile), which links the engine
// library; the reference's CLI, acceptance harness and unit suites are built
// against both.  Neither module is on the integration path.
#pragma once

#include <span>
#include <vector>

#include "fembatch_b200.hpp"

namespace fembatch {

// ---- verification (reference include/fembatch/oracle.hpp) ----------------
// An independent FP64 element matrix by direct quadrature in physical space
// (pulled-back P1 gradients per quadrature point; never G or K) and a store
// checker built on it, for callers that want to check results.  Host code;
// the integration and assembly paths never call it.
struct OracleReport {
  double max_rel_error = 0.0;  // |got - exact| / max(|exact|, 1e-14)
  double max_abs_error = 0.0;
  std::int64_t worst_element = -1;
  int worst_test_index = -1;
  int worst_trial_index = -1;
  double tolerance = 0.0;
  bool passed = false;
};
// Row-major krows x krows; vertex_coords (dim+1)*dim; coefficients: nb nodal
// values for the weighted form, empty otherwise (std::invalid_argument).
std::vector<double> assemble_element_direct(const FormSpec& spec, std::span<const double> vertex_coords,
                                            std::span<const double> coefficients = {});
OracleReport verify(const ElementMatrixStore& store, const Mesh& mesh, const FormSpec& spec,
                    const KernelConfig& config, const CoefficientField* coefficients, double tolerance);

// ---- benchmark runner (reference include/fembatch/bench.hpp) -------------
// run_benchmark times this engine's API calls (integrate_batches on the GPU,
// plus pack_geometry with include_packing) by wall clock, host data in and
// out, like the reference times its CPU engine.
struct BenchOptions {
  Operator op = Operator::laplacian;
  int dim = 3;
  int n = 16;  // structured mesh resolution
  double jitter = 0.0;
  std::uint64_t seed = 42;
  KernelConfig config;
  int workers = 1;
  int repetitions = 3;
  bool include_packing = false;
  bool verify_first = false;
};
// Axis values sorted and deduplicated; rows in lexicographic (bs, ce,
// interleave, unroll) order; invalid points become status rows.
struct SweepGrid {
  BenchOptions base;
  std::vector<int> batch_sizes{16, 32, 64, 128};
  std::vector<int> concurrent{1, 2, 4};
  std::vector<bool> interleave{false, true};
  std::vector<bool> unroll{false, true};
};
BenchRecord run_benchmark(const BenchOptions& options);
std::vector<BenchRecord> sweep(const SweepGrid& grid);

}  // namespace fembatch
