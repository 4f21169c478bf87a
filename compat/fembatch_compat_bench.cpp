// fembatch_compat_bench.cpp -- the reference's benchmark runner
// (include/fembatch/bench.hpp: run_benchmark, sweep) on the B200 engine, for
// the reference CLI and acceptance harness (compatibility library, not the
// product).  Behaviour contract taken from the reference's interface and
// tests (tests/test_bench.cpp, tests/acceptance.cpp criterion 8): a case is a
// structured (optionally jittered) mesh + form; each configuration is
// screened (invalid divisibility / work-group bound become status rows, not
// exceptions), optionally verified against the direct oracle first, then
// timed by wall clock over `repetitions` calls of the engine's API;
// gflops uses the best time and the paper's flop count; the checksum is that
// of the last store.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

#include "../include/fembatch_compat.hpp"

namespace fembatch {

namespace {

struct Case {
  FormSpec spec;
  AnalyticTensor k;
  Mesh mesh;
  CoefficientField w;
  const CoefficientField* coefficients() const { return spec.coefficient_arity == 1 ? &w : nullptr; }
};

Case build_case(const BenchOptions& o)
{
  Case c;
  c.spec = make_form_spec(o.op, o.dim);
  c.k = build_analytic_tensor(o.op, o.dim);
  c.mesh = structured_simplicial_mesh(o.dim, o.n);
  if (o.jitter > 0.0)
    c.mesh = jitter_mesh(c.mesh, o.jitter, o.seed);
  if (c.spec.coefficient_arity == 1)
    c.w = default_coefficient_field(c.mesh);
  return c;
}

// The record's identifying columns, as the options describe the run.
BenchRecord describe(const BenchOptions& o)
{
  BenchRecord r;
  r.op = operator_name(o.op);
  r.dim = o.dim;
  r.num_elements = o.dim == 2 ? 2LL * o.n * o.n : 6LL * o.n * o.n * o.n;
  r.batch_size = o.config.element_batch_size;
  r.concurrent = o.config.num_concurrent_elements;
  r.interleave = o.config.interleave_stores;
  r.unroll = o.config.loop_unroll;
  r.precision = precision_name(o.config.precision);
  r.workers = o.workers;
  r.reps = o.repetitions;
  r.status = "ok";
  return r;
}

// Status text of a configuration the engine would reject, "" if runnable.
std::string screen(const FormSpec& spec, const KernelConfig& c)
{
  const int bs = c.element_batch_size, ce = c.num_concurrent_elements;
  if (bs <= 0 || ce <= 0 || bs % ce != 0)
    return "invalid: divisibility";
  if (static_cast<std::int64_t>(spec.krows()) * spec.krows() * ce > work_group_bound)
    return "invalid: work-group bound";
  return "";
}

void verify_or_throw(const Case& cs, const KernelVariant& v, const KernelConfig& c, int workers)
{
  const ElementMatrixStore s = integrate_batches(v, pack_geometry(cs.mesh, c), cs.coefficients(), workers);
  const OracleReport rep = verify(s, cs.mesh, cs.spec, c, cs.coefficients(), default_tolerance(c.precision));
  if (rep.passed)
    return;
  char msg[192];
  std::snprintf(msg, sizeof msg, "verification failed: max relative error %.3e > %.3e at element %lld entry (%d, %d)",
                rep.max_rel_error, rep.tolerance, static_cast<long long>(rep.worst_element), rep.worst_test_index,
                rep.worst_trial_index);
  throw std::runtime_error(msg);
}

BenchRecord measure(const Case& cs, const BenchOptions& o)
{
  BenchRecord rec = describe(o);
  const KernelConfig& c = o.config;
  if (const std::string why = screen(cs.spec, c); !why.empty())
  {
    rec.status = why;
    return rec;
  }
  if (o.repetitions < 1)
    throw std::invalid_argument("repetition count must be >= 1");
  const KernelVariant v = specialize_kernel(cs.spec, cs.k, c);
  if (o.verify_first)
    verify_or_throw(cs, v, c, o.workers);

  // the timed call: mesh in -> matrices out (include_packing) or packed G in
  PackedGeometry packed;
  if (!o.include_packing)
    packed = pack_geometry(cs.mesh, c);
  ElementMatrixStore last;
  const std::function<void()> call = [&]
  {
    last = o.include_packing ? integrate_batches(v, pack_geometry(cs.mesh, c), cs.coefficients(), o.workers)
                             : integrate_batches(v, packed, cs.coefficients(), o.workers);
  };
  std::vector<double> seconds;
  seconds.reserve(o.repetitions);
  for (int i = 0; i < o.repetitions; ++i)
  {
    const auto t0 = std::chrono::steady_clock::now();
    call();
    seconds.push_back(std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
  }
  double sum = 0.0;
  for (double s : seconds)
    sum += s;
  rec.num_elements = cs.mesh.num_elements();
  rec.seconds_min = *std::min_element(seconds.begin(), seconds.end());
  rec.seconds_mean = sum / o.repetitions;
  rec.gflops = rec.seconds_min > 0.0
                   ? static_cast<double>(flop_count(cs.spec, c, rec.num_elements)) / rec.seconds_min * 1e-9
                   : 0.0;
  rec.checksum = store_checksum(last);
  return rec;
}

template <class T>
std::vector<T> axis(const std::vector<T>& values)
{
  std::vector<T> a(values);
  std::sort(a.begin(), a.end());
  a.erase(std::unique(a.begin(), a.end()), a.end());
  return a;
}

// Grid points in lexicographic (bs, ce, interleave, unroll) order.
std::vector<BenchOptions> grid_points(const SweepGrid& g)
{
  std::vector<BenchOptions> pts;
  const auto bss = axis(g.batch_sizes);
  const auto ces = axis(g.concurrent);
  const auto ils = axis(g.interleave);
  const auto urs = axis(g.unroll);
  pts.reserve(bss.size() * ces.size() * ils.size() * urs.size());
  for (int bs : bss)
    for (int ce : ces)
      for (bool il : ils)
        for (bool ur : urs)
        {
          BenchOptions o = g.base;
          o.config.element_batch_size = bs;
          o.config.num_concurrent_elements = ce;
          o.config.interleave_stores = il;
          o.config.loop_unroll = ur;
          pts.push_back(o);
        }
  return pts;
}

}  // namespace

BenchRecord run_benchmark(const BenchOptions& options) { return measure(build_case(options), options); }

std::vector<BenchRecord> sweep(const SweepGrid& grid)
{
  const Case cs = build_case(grid.base);
  std::vector<BenchRecord> rows;
  for (const BenchOptions& o : grid_points(grid))
  {
    try
    {
      rows.push_back(measure(cs, o));
    }
    catch (const std::exception& e)  // a failing point is a row, the sweep goes on
    {
      BenchRecord r = describe(o);
      r.status = std::string("error: ") + e.what();
      rows.push_back(std::move(r));
    }
  }
  return rows;
}

}  // namespace fembatch
