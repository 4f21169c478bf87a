// test_api.cpp -- the reference-compatible C++ API (include/fembatch_b200.hpp)
// exercised the way the reference's own doctest suites exercise fembatch
// (tests/test_engine.cpp, test_geometry.cpp, test_forms.cpp).  doctest is not
// available in this image, so a minimal CHECK harness stands in.
//
//   test_api cpu   -- host-only cases (forms, mesh synthesis, layouts, validation)
//   test_api all   -- plus the GPU integration cases (needs a CUDA device)
#include <cmath>
#include <cstdio>
#include <fstream>
#include <iterator>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "fembatch_b200.hpp"

using namespace fembatch;

namespace {

int g_failures = 0, g_checks = 0;
const char* g_case = "";

#define CHECK(cond)                                                                   \
  do                                                                                  \
  {                                                                                   \
    ++g_checks;                                                                       \
    if (!(cond))                                                                      \
    {                                                                                 \
      ++g_failures;                                                                   \
      std::printf("  FAIL [%s] %s:%d: %s\n", g_case, __FILE__, __LINE__, #cond);      \
    }                                                                                 \
  } while (0)

template <class E, class F>
bool throws_as(F&& f, const char* contains = nullptr)
{
  try
  {
    f();
  }
  catch (const E& e)
  {
    return contains == nullptr || std::strstr(e.what(), contains) != nullptr;
  }
  catch (...)
  {
    return false;
  }
  return false;
}

#define CHECK_THROWS_AS(expr, E) CHECK(throws_as<E>([&] { (void)(expr); }))
#define CHECK_THROWS_WITH_AS(expr, text, E) CHECK(throws_as<E>([&] { (void)(expr); }, text))

struct Case {
  const char* name;
  bool gpu;
  std::function<void()> fn;
};
std::vector<Case>& cases()
{
  static std::vector<Case> c;
  return c;
}
struct Reg {
  Reg(const char* n, bool gpu, std::function<void()> f) { cases().push_back({n, gpu, std::move(f)}); }
};
#define TEST_CASE(name, gpu) static void name(); static Reg reg_##name(#name, gpu, name); static void name()

KernelConfig config_of(int bs, int ce, bool is, bool ur, Precision p)
{
  KernelConfig c;
  c.element_batch_size = bs;
  c.num_concurrent_elements = ce;
  c.interleave_stores = is;
  c.loop_unroll = ur;
  c.precision = p;
  return c;
}

Mesh reference_element_mesh(int dim, int copies = 1)
{
  Mesh m;
  m.dim = dim;
  m.vertices = dim == 2 ? std::vector<double>{0, 0, 1, 0, 0, 1}
                        : std::vector<double>{0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0, 1};
  for (int c = 0; c < copies; ++c)
    for (int k = 0; k <= dim; ++k)
      m.cells.push_back(k);
  return m;
}

// the reference library composition (tests/test_engine.cpp:28-38), on the GPU
ElementMatrixStore integrate(Operator op, const Mesh& mesh, const KernelConfig& config,
                             const CoefficientField* w = nullptr, int workers = 1)
{
  const FormSpec spec = make_form_spec(op, mesh.dim);
  const AnalyticTensor k = build_analytic_tensor(op, mesh.dim);
  const KernelVariant variant = specialize_kernel(spec, k, config);
  const PackedGeometry geom = pack_geometry(mesh, config);
  return integrate_batches(variant, geom, w, workers);
}

const double ref_tri[3][3] = {{1.0, -0.5, -0.5}, {-0.5, 0.5, 0.0}, {-0.5, 0.0, 0.5}};

// ------------------------------------------------------------------ host cases
TEST_CASE(element_matrix_indexing, false)
{
  CHECK(element_matrix_index(3, 4, 2, 3, 0, 0) == 1 * (2 * 9) + 1 * 9);
  CHECK(element_matrix_index(3, 4, 2, 3, 2, 1) == 1 * (2 * 9) + 1 * 9 + 2 + 1 * 3);
  CHECK(element_matrix_index(3, 1, 1, 0, 1, 2) == 1 + 2 * 3);
  CHECK(element_matrix_index(3, 1, 1, 2, 0, 0) == 2 * 9);
}

TEST_CASE(specialization_contract, false)
{
  const FormSpec spec = make_form_spec(Operator::laplacian, 3);
  const AnalyticTensor k = build_analytic_tensor(Operator::laplacian, 3);
  CHECK_THROWS_AS(specialize_kernel(spec, k, config_of(5, 2, false, false, Precision::f64)), std::invalid_argument);
  CHECK_THROWS_AS(specialize_kernel(spec, k, config_of(0, 1, false, false, Precision::f64)), std::invalid_argument);
  const FormSpec el = make_form_spec(Operator::elasticity, 3);
  const AnalyticTensor ke = build_analytic_tensor(Operator::elasticity, 3);
  CHECK_THROWS_WITH_AS(specialize_kernel(el, ke, config_of(64, 8, false, false, Precision::f64)),
                       "work-group bound", std::invalid_argument);
  CHECK(specialize_kernel(el, ke, config_of(64, 4, false, false, Precision::f64)).description == "bs64_ce4");
  CHECK_THROWS_AS(specialize_kernel(el, k, config_of(64, 1, false, false, Precision::f64)), std::invalid_argument);
  CHECK(specialize_kernel(spec, k, config_of(128, 2, true, false, Precision::f32)).description == "bs128_ce2_is");
  CHECK(specialize_kernel(spec, k, config_of(16, 4, false, true, Precision::f64)).description == "bs16_ce4_unroll");
  CHECK(specialize_kernel(spec, k, config_of(32, 1, true, true, Precision::f64)).description
        == "bs32_ce1_is_unroll");
}

TEST_CASE(analytic_tensor_goldens, false)
{
  // reference tests/test_forms.cpp:49-133
  const AnalyticTensor k2 = build_k_laplacian(2);
  for (int t = 0; t < 4; ++t)
    CHECK(k2.blocks[t] == 0.5);
  CHECK(k2.block_offset(1, 2) == 28);
  CHECK(k2.entry(1, 2, 0, 0, 1) == 0.5 && k2.entry(1, 2, 0, 0, 0) == 0.0);
  CHECK(build_k_weighted_laplacian(2).block_offset(1, 2, 2) == 92);
  CHECK(build_k_laplacian(3).entry(1, 1, 0, 0, 0) == 1.0 / 6.0);
  for (int dim : {2, 3})
  {
    const AnalyticTensor kl = build_k_laplacian(dim), ke = build_k_elasticity(dim);
    const int nb = dim + 1;
    bool ok = true;
    for (int a = 0; a < nb; ++a)
      for (int b = 0; b < nb; ++b)
        for (int c = 0; c < dim; ++c)
          for (int d = 0; d < dim; ++d)
            for (int mu = 0; mu < dim; ++mu)
              for (int nu = 0; nu < dim; ++nu)
              {
                const double got = ke.entry(a + c * nb, b + d * nb, 0, mu, nu);
                const double want = c == d ? 0.25 * kl.entry(a, b, 0, mu, nu) : 0.0;
                ok = ok && std::memcmp(&got, &want, sizeof got) == 0;
              }
    CHECK(ok);
  }
}

TEST_CASE(jacobian_and_geometry_goldens, false)
{
  // reference tests/test_geometry.cpp:117-194
  Mesh tri = reference_element_mesh(2);
  ElementJacobian jac = element_jacobian(tri, 0);
  CHECK(jac.j[0] == 1.0 && jac.j[1] == 0.0 && jac.j[2] == 0.0 && jac.j[3] == 1.0 && jac.det == 1.0);
  tri.vertices = {0.0, 0.0, 1.0, 0.0, 1.0, 1.0};
  GeometryTensor g = geometry_tensor(element_jacobian(tri, 0));
  CHECK(g.entry(0, 0) == 2.0 && g.entry(0, 1) == -1.0 && g.entry(1, 0) == -1.0 && g.entry(1, 1) == 1.0);
  Mesh bad = reference_element_mesh(2);
  bad.cells = {0, 2, 1};
  CHECK_THROWS_WITH_AS(element_jacobian(bad, 0), "cell 0", std::runtime_error);
  CHECK_THROWS_AS(element_jacobian(bad, 5), std::out_of_range);
  double degenerate[6] = {0.0, 0.0, 1.0, 1.0, 2.0, 2.0};
  CHECK_THROWS_AS(jacobian_from_vertices(2, degenerate), std::runtime_error);
  CHECK(packed_geometry_index(2, 5, 1, 0, 1, 0) == 22);
  CHECK(packed_geometry_index(3, 128, 2, 1, 2, 1) == 2 * 9 * 128 + 9 + 7);
}

TEST_CASE(mesh_synthesis_and_io, false)
{
  const Mesh s = structured_simplicial_mesh(3, 2);
  CHECK(s.num_elements() == 48 && s.num_vertices() == 27);
  for (std::int64_t e = 0; e < s.num_elements(); ++e)
    CHECK(element_jacobian(s, e).det > 0.0);
  const Mesh j = jitter_mesh(structured_simplicial_mesh(2, 3), 0.15, 13);
  std::stringstream ss;
  write_mesh_text(ss, j);
  const Mesh back = read_mesh_text(ss);
  CHECK(back.vertices == j.vertices && back.cells == j.cells);
  CHECK_THROWS_AS(jitter_mesh(s, 0.25, 42), std::invalid_argument);
  Mesh m = reference_element_mesh(2);
  m.cells[2] = 9;
  CHECK_THROWS_AS(validate_mesh(m), std::invalid_argument);
}

TEST_CASE(flop_count_rule, false)
{
  const KernelConfig c;
  CHECK(flop_count(make_form_spec(Operator::laplacian, 3), c, 1) == 288);
  CHECK(flop_count(make_form_spec(Operator::elasticity, 2), c, 1) == 288);
  CHECK(flop_count(make_form_spec(Operator::weighted_laplacian, 2), c, 1) == 270);
  CHECK(flop_count(make_form_spec(Operator::laplacian, 2), c, 10) == 720);
}

// ------------------------------------------------------------------- GPU cases
TEST_CASE(reference_triangle_is_exact, true)
{
  const ElementMatrixStore s = integrate(Operator::laplacian, reference_element_mesh(2),
                                         config_of(1, 1, false, false, Precision::f64));
  const std::vector<double> m = unpack_element_matrix(s, config_of(1, 1, false, false, Precision::f64),
                                                      make_form_spec(Operator::laplacian, 2), 0);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      CHECK(m[i * 3 + j] == ref_tri[i][j]);
}

TEST_CASE(variant_and_worker_invariance_bitwise, true)
{
  const Mesh mesh = jitter_mesh(structured_simplicial_mesh(2, 4), 0.15, 42);
  for (Precision p : {Precision::f64, Precision::f32})
  {
    const KernelConfig base = config_of(16, 1, false, false, p);
    const ElementMatrixStore ref = integrate(Operator::laplacian, mesh, base);
    const FormSpec spec = make_form_spec(Operator::laplacian, 2);
    for (int bs : {16, 32})
      for (int ce : {1, 2, 4})
        for (bool is : {false, true})
          for (bool ur : {false, true})
            for (int workers : {1, 3})
            {
              const KernelConfig c = config_of(bs, ce, is, ur, p);
              const ElementMatrixStore got = integrate(Operator::laplacian, mesh, c, nullptr, workers);
              bool same = true;
              for (std::int64_t e = 0; e < mesh.num_elements(); ++e)
                same = same && unpack_element_matrix(ref, base, spec, e) == unpack_element_matrix(got, c, spec, e);
              CHECK(same);
            }
  }
}

TEST_CASE(fused_mesh_path_equals_pack_plus_integrate, true)
{
  for (Operator op : {Operator::laplacian, Operator::elasticity, Operator::weighted_laplacian})
    for (int dim : {2, 3})
      for (Precision p : {Precision::f32, Precision::f64})
      {
        const Mesh mesh = jitter_mesh(structured_simplicial_mesh(dim, dim == 2 ? 9 : 3), 0.15, 42);
        CoefficientField w;
        const CoefficientField* wp = nullptr;
        if (op == Operator::weighted_laplacian)
        {
          w.num_basis_funcs = dim + 1;
          for (std::int64_t e = 0; e < mesh.num_elements(); ++e)
            for (int k = 0; k <= dim; ++k)
              w.values.push_back(1.0 + mesh.vertex(mesh.cell_vertex(e, k), 0));
          wp = &w;
        }
        const KernelConfig c = config_of(16, 2, true, false, p);
        const FormSpec spec = make_form_spec(op, dim);
        const KernelVariant v = specialize_kernel(spec, build_analytic_tensor(op, dim), c);
        const ElementMatrixStore a = integrate_batches(v, pack_geometry(mesh, c), wp);
        const ElementMatrixStore b = integrate_mesh(v, mesh, wp);
        CHECK(scalar_array_size(a.data) == scalar_array_size(b.data));
        bool same = true;
        for (std::int64_t t = 0; t < scalar_array_size(a.data); ++t)
        {
          const double x = scalar_array_at(a.data, t), y = scalar_array_at(b.data, t);
          same = same && std::memcmp(&x, &y, sizeof x) == 0;
        }
        CHECK(same);
      }
}

TEST_CASE(null_spaces_and_symmetry, true)
{
  const Mesh mesh = jitter_mesh(structured_simplicial_mesh(3, 3), 0.15, 42);
  const KernelConfig c = config_of(32, 4, false, true, Precision::f64);
  const ElementMatrixStore s = integrate(Operator::laplacian, mesh, c);
  const FormSpec spec = make_form_spec(Operator::laplacian, 3);
  double worst = 0.0;
  for (std::int64_t e = 0; e < mesh.num_elements(); ++e)
  {
    const std::vector<double> m = unpack_element_matrix(s, c, spec, e);
    for (int i = 0; i < 4; ++i)
    {
      double row = 0.0;
      for (int j = 0; j < 4; ++j)
      {
        row += m[i * 4 + j];
        CHECK(m[i * 4 + j] == m[j * 4 + i]);
      }
      worst = std::max(worst, std::abs(row));
    }
  }
  CHECK(worst <= 1e-12);
}

TEST_CASE(synthetic_scaled_identity_geometry, true)
{
  // reference tests/test_engine.cpp:337-378
  PackedGeometry geom;
  geom.dim = 2;
  geom.element_batch_size = 4;
  geom.num_batches = 2;
  geom.num_elements = 5;
  geom.precision = Precision::f64;
  geom.data = make_scalar_array(Precision::f64, 2 * 4 * 4);
  auto& d = std::get<std::vector<double>>(geom.data);
  for (int slot = 0; slot < 8; ++slot)
  {
    const double c = slot < 5 ? slot + 1.0 : 7.5;
    d[slot * 4 + 0] = d[slot * 4 + 3] = c;
  }
  const KernelConfig c = config_of(4, 2, true, true, Precision::f64);
  const FormSpec spec = make_form_spec(Operator::laplacian, 2);
  const ElementMatrixStore s = integrate_batches(specialize_kernel(spec, build_k_laplacian(2), c), geom);
  CHECK(scalar_array_size(s.data) == 72);
  for (int e = 0; e < 5; ++e)
  {
    const std::vector<double> m = unpack_element_matrix(s, c, spec, e);
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j)
        CHECK(m[i * 3 + j] == (e + 1) * ref_tri[i][j]);
  }
}

TEST_CASE(input_validation_and_errors, true)
{
  const Mesh mesh = structured_simplicial_mesh(2, 2);
  const KernelConfig c = config_of(8, 1, false, false, Precision::f64);
  const KernelVariant wv = specialize_kernel(make_form_spec(Operator::weighted_laplacian, 2),
                                             build_k_weighted_laplacian(2), c);
  const PackedGeometry geom = pack_geometry(mesh, c);
  CHECK_THROWS_AS(integrate_batches(wv, geom, nullptr), std::invalid_argument);
  const KernelVariant lv = specialize_kernel(make_form_spec(Operator::laplacian, 2), build_k_laplacian(2), c);
  KernelConfig other = c;
  other.element_batch_size = 16;
  CHECK_THROWS_AS(integrate_batches(lv, pack_geometry(mesh, other), nullptr), std::invalid_argument);
  KernelConfig single = c;
  single.precision = Precision::f32;
  CHECK_THROWS_AS(integrate_batches(lv, pack_geometry(mesh, single), nullptr), std::invalid_argument);
  CHECK_THROWS_AS(integrate_batches(lv, geom, nullptr, 0), std::invalid_argument);
  Mesh bad = mesh;
  std::swap(bad.cells[3 * 3 + 1], bad.cells[3 * 3 + 2]);  // invert cell 3
  CHECK_THROWS_WITH_AS(pack_geometry(bad, c), "degenerate element: det(J) <= 0 in cell 3", std::runtime_error);
  CHECK_THROWS_WITH_AS(integrate_mesh(lv, bad), "in cell 3", std::runtime_error);
}

TEST_CASE(store_round_trip, true)
{
  const Mesh mesh = jitter_mesh(structured_simplicial_mesh(2, 3), 0.15, 17);
  for (Precision p : {Precision::f64, Precision::f32})
  {
    const KernelConfig c = config_of(8, 2, false, false, p);
    const ElementMatrixStore s = integrate(Operator::laplacian, mesh, c);
    std::stringstream ss;
    write_store(ss, s);
    const ElementMatrixStore back = read_store(ss);
    CHECK(back.num_elements == s.num_elements && back.num_batches == s.num_batches && back.precision == s.precision);
    bool same = scalar_array_size(back.data) == scalar_array_size(s.data);
    for (std::int64_t t = 0; same && t < scalar_array_size(s.data); ++t)
      same = scalar_array_at(back.data, t) == scalar_array_at(s.data, t);
    CHECK(same);
  }
  std::stringstream junk("not a store file at all");
  CHECK_THROWS_AS(read_store(junk), std::runtime_error);
}

std::string g_golden = "tests/golden";  // argv[2]: the golden-file directory

std::string slurp(const std::string& path)
{
  std::ifstream f(path, std::ios::binary);
  return std::string(std::istreambuf_iterator<char>(f), std::istreambuf_iterator<char>());
}

struct RefFile {
  const char* name;
  Operator op;
  int bs, ce;
  Precision p;
};
const RefFile kRefFiles[] = {{"ref_store_2d_elasticity_f32", Operator::elasticity, 8, 2, Precision::f32},
                             {"ref_store_3d_laplacian_f64", Operator::laplacian, 16, 1, Precision::f64}};

// F4 formats against files the UNMODIFIED reference wrote
// (tests/golden/make_golden.py): FBEMAT01 store (src/engine.cpp:413-508) and
// text mesh (src/geometry.cpp:353-395) read back and re-written byte for byte.
TEST_CASE(reference_written_files_round_trip, false)
{
  for (const RefFile& f : kRefFiles)
  {
    const std::string sbytes = slurp(g_golden + "/" + f.name + ".fbemat");
    const std::string mtext = slurp(g_golden + "/" + f.name + ".mesh");
    CHECK(!sbytes.empty() && !mtext.empty());
    std::istringstream si(sbytes);
    const ElementMatrixStore s = read_store(si);
    CHECK(s.precision == f.p && s.element_batch_size == f.bs && s.num_concurrent_elements == f.ce);
    std::ostringstream so;
    write_store(so, s);
    CHECK(so.str() == sbytes);
    std::istringstream mi(mtext);
    const Mesh m = read_mesh_text(mi);
    CHECK(s.num_elements == m.num_elements() && s.dim == m.dim);
    std::ostringstream mo;
    write_mesh_text(mo, m);
    CHECK(mo.str() == mtext);
  }
}

// ... and the GPU engine reproduces the reference's store file exactly from
// the reference's mesh file.
TEST_CASE(gpu_store_equals_reference_file_bytes, true)
{
  for (const RefFile& f : kRefFiles)
  {
    std::istringstream mi(slurp(g_golden + "/" + f.name + ".mesh"));
    const Mesh m = read_mesh_text(mi);
    const ElementMatrixStore s = integrate(f.op, m, config_of(f.bs, f.ce, true, false, f.p));
    std::ostringstream so;
    write_store(so, s);
    CHECK(so.str() == slurp(g_golden + "/" + f.name + ".fbemat"));
  }
}

TEST_CASE(assembly_plan_pattern_and_validation, false)
{
  const Mesh mesh = structured_simplicial_mesh(2, 2);  // 9 vertices, 8 triangles
  const AssemblyPlan lap = make_assembly_plan(Operator::laplacian, mesh);
  CHECK(lap.rows == 9);
  const AssemblyPlan el = make_assembly_plan(Operator::elasticity, mesh);
  CHECK(el.rows == 18 && el.nnz == 4 * lap.nnz);
  Mesh bad = mesh;
  bad.cells[4] = 99;  // cell 1
  CHECK_THROWS_WITH_AS(make_assembly_plan(Operator::laplacian, bad), "out of range in cell 1", std::invalid_argument);
  bad = mesh;
  bad.cells[5] = bad.cells[3];  // cell 1 repeats a vertex
  CHECK_THROWS_WITH_AS(make_assembly_plan(Operator::laplacian, bad), "repeated vertex in cell 1",
                       std::invalid_argument);
}

// F4 bench records against the reference CLI's own sweep table
// (tests/golden/ref_bench_sweep.csv): read back and re-written byte for byte;
// the JSON form of the same records goes to $FB_TEST_JSON_OUT when set
// (tests/test_cpp_api.py compares it with the Python writer, which is pinned
// to the reference's JSON bytes), and the reader rejects malformed tables.
TEST_CASE(bench_records_round_trip, false)
{
  const std::string csv = slurp(g_golden + "/ref_bench_sweep.csv");
  CHECK(!csv.empty());
  std::istringstream in(csv);
  const std::vector<BenchRecord> recs = read_csv(in);
  CHECK(recs.size() == 16 && recs[0].op == "laplacian" && recs[4].status == "invalid: divisibility");
  std::ostringstream out;
  write_csv(out, recs);
  CHECK(out.str() == csv);
  if (const char* path = std::getenv("FB_TEST_JSON_OUT"))
  {
    std::ofstream f(path, std::ios::binary);
    write_json(f, recs);
  }
  for (const char* bad : {"", "wrong,header\n", "operator,dim,num_elements,batch_size,concurrent,interleave,unroll,"
                                                 "precision,workers,reps,seconds_min,seconds_mean,gflops,checksum,"
                                                 "status\n\"laplacian\",2\n"})
  {
    std::istringstream b(bad);
    CHECK_THROWS_AS(read_csv(b), std::runtime_error);
  }
  CHECK(default_tolerance(Precision::f64) == 1e-12 && default_tolerance(Precision::f32) == 5e-5);
}

TEST_CASE(global_assembly_is_the_serial_element_sum, true)
{
  const Mesh mesh = jitter_mesh(structured_simplicial_mesh(3, 3), 0.15, 42);
  for (Precision p : {Precision::f64, Precision::f32})
    for (Operator op : {Operator::laplacian, Operator::elasticity})
    {
      const KernelConfig c = config_of(16, 1, false, false, p);
      const ElementMatrixStore s = integrate(op, mesh, c);
      const FormSpec spec = make_form_spec(op, 3);
      const KernelVariant v = specialize_kernel(spec, build_analytic_tensor(op, 3), c);
      const AssemblyPlan plan = make_assembly_plan(op, mesh);
      const CsrMatrix a = assemble_global(v, plan, s, true);
      const CsrMatrix b = assemble_global(v, plan, s, false);
      CHECK(a.rows == plan.rows && static_cast<std::int64_t>(a.col_idx.size()) == plan.nnz);
      // serial element-order sum in engine precision (the definition)
      const int nc = op == Operator::elasticity ? 3 : 1, kr = spec.krows();
      std::vector<double> want(plan.nnz, 0.0);
      std::vector<float> want32(plan.nnz, 0.0f);
      for (std::int64_t e = 0; e < mesh.num_elements(); ++e)
        for (int j = 0; j < kr; ++j)
          for (int i = 0; i < kr; ++i)
          {
            const std::int64_t row = std::int64_t(mesh.cells[e * 4 + i % 4]) * nc + i / 4;
            const std::int32_t col = mesh.cells[e * 4 + j % 4] * nc + j / 4;
            std::int64_t z = a.row_ptr[row];
            while (a.col_idx[z] != col)
              ++z;
            const double x = scalar_array_at(s.data, e * kr * kr + i + std::int64_t(j) * kr);
            if (p == Precision::f64)
              want[z] = want[z] + x;
            else
              want32[z] = want32[z] + static_cast<float>(x);
          }
      bool same = true;
      for (std::int64_t z = 0; same && z < plan.nnz; ++z)
      {
        const double w = p == Precision::f64 ? want[z] : double(want32[z]);
        same = scalar_array_at(a.values, z) == w && scalar_array_at(b.values, z) == w;
      }
      CHECK(same);
      // the same operator straight from packed geometry (no element store)
      const PackedGeometry geom = pack_geometry(mesh, c);
      const CsrMatrix g = assemble_global(v, plan, geom);
      const CsrMatrix gs = assemble_global(v, plan, integrate_batches(v, geom));
      bool gsame = g.values.index() == gs.values.index();
      for (std::int64_t z = 0; gsame && z < plan.nnz; ++z)
        gsame = scalar_array_at(g.values, z) == scalar_array_at(gs.values, z) &&
                scalar_array_at(g.values, z) == scalar_array_at(a.values, z);
      CHECK(gsame);
    }
}

}  // namespace

int main(int argc, char** argv)
{
  const bool gpu = argc > 1 && std::strcmp(argv[1], "all") == 0;
  if (argc > 2)
    g_golden = argv[2];
  int ran = 0;
  for (const Case& c : cases())
  {
    if (c.gpu && !gpu)
      continue;
    g_case = c.name;
    const int before = g_failures;
    try
    {
      c.fn();
    }
    catch (const std::exception& e)
    {
      ++g_failures;
      std::printf("  FAIL [%s] unexpected exception: %s\n", c.name, e.what());
    }
    std::printf("[%s] %s\n", g_failures == before ? "PASS" : "FAIL", c.name);
    ++ran;
  }
  std::printf("%d cases, %d checks, %d failures\n", ran, g_checks, g_failures);
  return g_failures == 0 ? 0 : 1;
}
