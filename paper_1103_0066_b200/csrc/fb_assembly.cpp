// fb_assembly.cpp -- extern "C" global assembly (include/fembatch_b200.h,
// "global assembly"): the plan (CSR pattern + vertex->element incidence
// lists, built once per mesh -- on the GPU for device-resident connectivity
// (fb_plan.cu), else on the host, multithreaded; the two are array-for-array
// identical) and the launch of the deterministic gather kernel
// (fb_assemble.cu).
//
// Plan construction:
//   1. incidences by counting sort over elements in ascending order, so each
//      vertex's list is ascending in e (this order IS the summation order);
//   2. per vertex, the sorted unique vertices of its incident elements (the
//      row block's columns);
//   3. per incidence, the neighbour slot of each of the element's vertices.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

#include "fb_capi_util.h"
#include "fb_internal.h"

using namespace fbc;

namespace {

// host connectivity from this size on is planned on the GPU (FB_PLAN_HOST in
// the environment forces the host builder)
constexpr int64_t kGpuPlanMinElements = 1 << 16;

struct DevPlan {
  int64_t* goff = nullptr;
  uint32_t* spk = nullptr;
  uint32_t* spos = nullptr;
  int64_t* nbr_ptr = nullptr;
  int32_t* nbr = nullptr;  // only on the device that built the plan
};

}  // namespace

struct fb_assembly {
  int op = 0, dim = 2, nb = 3, nc = 1;
  int64_t nv = 0, ne = 0;
  std::vector<int64_t> v2e_ptr, nbr_ptr;  // nv + 1 each
  std::vector<uint32_t> v2e;              // e << 2 | a, ascending e per vertex
  std::vector<uint8_t> nbrpos;            // nb per incidence
  std::vector<int32_t> nbr;               // sorted neighbour vertices per vertex
  // device layout (SELL-32, fb_internal.h AsmArgs)
  std::vector<int64_t> goff;
  std::vector<uint32_t> spk, spos;
  int64_t total_nbr = 0;  // sum of vertex degrees
  int home = -1;          // device that built the plan (host arrays filled lazily), -1 = host-built
  mutable std::mutex mu;
  mutable std::map<int, DevPlan> dev;
  int64_t rows() const { return nv * nc; }
  int64_t nnz() const { return total_nbr * nc * nc; }
  ~fb_assembly()
  {
    int cur = 0;
    cudaGetDevice(&cur);
    for (auto& [d, p] : dev)
    {
      cudaSetDevice(d);
      cudaFree(p.goff);
      cudaFree(p.spk);
      cudaFree(p.spos);
      cudaFree(p.nbr_ptr);
      cudaFree(p.nbr);
    }
    cudaSetDevice(cur);
  }
};

namespace {

template <class F>
void parallel_for(int64_t n, F&& f)
{
  const int64_t hw = std::max(1u, std::thread::hardware_concurrency());
  const int64_t nt = std::min<int64_t>(hw, std::max<int64_t>(1, n / 4096));
  if (nt <= 1)
  {
    f(0, n, 0);
    return;
  }
  std::vector<std::thread> th;
  for (int64_t t = 0; t < nt; ++t)
    th.emplace_back([&, t] { f(n * t / nt, n * (t + 1) / nt, static_cast<int>(t)); });
  for (auto& x : th)
    x.join();
}

void build_plan(fb_assembly& A, const int32_t* cells)
{
  const int nb = A.nb;
  const int64_t nv = A.nv, ne = A.ne;
  // validation (first offending cell in element order)
  for (int64_t e = 0; e < ne; ++e)
    for (int a = 0; a < nb; ++a)
    {
      const int32_t v = cells[e * nb + a];
      if (v < 0 || v >= nv)
        throw_code(FB_ERR_INVALID_ARGUMENT, "cell vertex index out of range in cell " + std::to_string(e), e);
      for (int b = 0; b < a; ++b)
        if (cells[e * nb + b] == v)
          throw_code(FB_ERR_INVALID_ARGUMENT, "repeated vertex in cell " + std::to_string(e), e);
    }
  // 1. incidences, ascending e per vertex
  A.v2e_ptr.assign(nv + 1, 0);
  for (int64_t i = 0; i < ne * nb; ++i)
    A.v2e_ptr[cells[i] + 1]++;
  for (int64_t v = 0; v < nv; ++v)
    A.v2e_ptr[v + 1] += A.v2e_ptr[v];
  A.v2e.resize(ne * nb);
  {
    std::vector<int64_t> fill(A.v2e_ptr.begin(), A.v2e_ptr.end() - 1);
    for (int64_t e = 0; e < ne; ++e)
      for (int a = 0; a < nb; ++a)
        A.v2e[fill[cells[e * nb + a]]++] = static_cast<uint32_t>(e << 2 | a);
  }
  // 2. neighbour lists (per thread chunk, then concatenated)
  std::vector<std::vector<int32_t>> chunk_nbr(std::max(1u, std::thread::hardware_concurrency()));
  std::vector<int64_t> deg(nv, 0);
  std::vector<int64_t> chunk_lo(chunk_nbr.size(), -1);
  parallel_for(nv,
               [&](int64_t v0, int64_t v1, int t)
               {
                 std::vector<int32_t> tmp;
                 auto& out = chunk_nbr[t];
                 chunk_lo[t] = v0;
                 for (int64_t v = v0; v < v1; ++v)
                 {
                   tmp.clear();
                   for (int64_t q = A.v2e_ptr[v]; q < A.v2e_ptr[v + 1]; ++q)
                   {
                     const int64_t e = A.v2e[q] >> 2;
                     for (int b = 0; b < nb; ++b)
                       tmp.push_back(cells[e * nb + b]);
                   }
                   std::sort(tmp.begin(), tmp.end());
                   tmp.erase(std::unique(tmp.begin(), tmp.end()), tmp.end());
                   deg[v] = static_cast<int64_t>(tmp.size());
                   out.insert(out.end(), tmp.begin(), tmp.end());
                 }
               });
  A.nbr_ptr.assign(nv + 1, 0);
  for (int64_t v = 0; v < nv; ++v)
  {
    if (deg[v] > 255)
      throw_code(FB_ERR_INVALID_ARGUMENT, "vertex degree exceeds 255 at vertex " + std::to_string(v), -1);
    A.nbr_ptr[v + 1] = A.nbr_ptr[v] + deg[v];
  }
  A.nbr.resize(A.nbr_ptr[nv]);
  A.total_nbr = A.nbr_ptr[nv];
  {
    std::vector<std::pair<int64_t, size_t>> order;
    for (size_t t = 0; t < chunk_nbr.size(); ++t)
      if (chunk_lo[t] >= 0)
        order.push_back({chunk_lo[t], t});
    std::sort(order.begin(), order.end());
    for (auto& [lo, t] : order)
      std::copy(chunk_nbr[t].begin(), chunk_nbr[t].end(), A.nbr.begin() + A.nbr_ptr[lo]);
  }
  if (A.nbr_ptr[nv] * A.nc > INT32_MAX || A.rows() > INT32_MAX)
    throw_code(FB_ERR_INVALID_ARGUMENT, "assembled operator exceeds 32-bit column indices", -1);
  // 3. neighbour slot of every local vertex of every incidence
  A.nbrpos.resize(ne * nb * nb);
  parallel_for(nv,
               [&](int64_t v0, int64_t v1, int)
               {
                 for (int64_t v = v0; v < v1; ++v)
                 {
                   const int32_t* lo = A.nbr.data() + A.nbr_ptr[v];
                   const int32_t* hi = A.nbr.data() + A.nbr_ptr[v + 1];
                   for (int64_t q = A.v2e_ptr[v]; q < A.v2e_ptr[v + 1]; ++q)
                   {
                     const int64_t e = A.v2e[q] >> 2;
                     for (int b = 0; b < nb; ++b)
                       A.nbrpos[q * nb + b] =
                           static_cast<uint8_t>(std::lower_bound(lo, hi, cells[e * nb + b]) - lo);
                   }
                 }
               });
  // 4. sliced (SELL-32) copy for coalesced warp loads: incidence k of vertex
  //    32g + l at goff[g] + 32k + l
  const int64_t ngroups = (nv + 31) / 32;
  A.goff.assign(ngroups + 1, 0);
  for (int64_t g = 0; g < ngroups; ++g)
  {
    int64_t w = 0;
    for (int64_t v = g * 32; v < std::min(nv, g * 32 + 32); ++v)
      w = std::max(w, A.v2e_ptr[v + 1] - A.v2e_ptr[v]);
    A.goff[g + 1] = A.goff[g] + 32 * w;
  }
  A.spk.assign(A.goff[ngroups], 0xffffffffu);
  A.spos.assign(A.goff[ngroups], 0u);
  parallel_for(ngroups,
               [&](int64_t g0, int64_t g1, int)
               {
                 for (int64_t g = g0; g < g1; ++g)
                   for (int64_t v = g * 32; v < std::min(nv, g * 32 + 32); ++v)
                     for (int64_t q = A.v2e_ptr[v]; q < A.v2e_ptr[v + 1]; ++q)
                     {
                       const int64_t at = A.goff[g] + 32 * (q - A.v2e_ptr[v]) + (v - g * 32);
                       A.spk[at] = A.v2e[q];
                       uint32_t w = 0;
                       for (int b = 0; b < nb; ++b)
                         w |= static_cast<uint32_t>(A.nbrpos[q * nb + b]) << (8 * b);
                       A.spos[at] = w;
                     }
               });
}

void build_plan_gpu(fb_assembly& A, const int32_t* cells, int dev)
{
  int cur = 0;
  cuda_check(cudaGetDevice(&cur), "cudaGetDevice");
  cuda_check(cudaSetDevice(dev), "cudaSetDevice");
  cudaStream_t st = nullptr;
  cuda_check(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "cudaStreamCreate");
  fbk::PlanDevice P;
  int64_t bad[3];
  const cudaError_t e = fbk::build_plan_device(A.dim, A.ne, A.nv, cells, st, &P, bad);
  cudaStreamDestroy(st);
  cudaSetDevice(cur);
  cuda_check(e, "assembly plan build");
  DevPlan p;
  p.goff = P.goff;
  p.spk = P.spk;
  p.spos = P.spos;
  p.nbr_ptr = P.nbr_ptr;
  p.nbr = P.nbr;
  if (bad[0] >= 0 || bad[1] >= 0)
  {
    // the lowest offending cell, and its failure reported exactly as the
    // host builder would (first bad slot in slot order): its ids are
    // rechecked on the host
    const int64_t c = bad[0] < 0 ? bad[1] : (bad[1] < 0 ? bad[0] : std::min(bad[0], bad[1]));
    int32_t ids[4] = {0, 0, 0, 0};
    cuda_check(cudaMemcpy(ids, cells + c * A.nb, A.nb * sizeof(int32_t), cudaMemcpyDefault), "download cell");
    for (int a = 0; a < A.nb; ++a)
    {
      if (ids[a] < 0 || ids[a] >= A.nv)
        throw_code(FB_ERR_INVALID_ARGUMENT, "cell vertex index out of range in cell " + std::to_string(c), c);
      for (int b = 0; b < a; ++b)
        if (ids[b] == ids[a])
          throw_code(FB_ERR_INVALID_ARGUMENT, "repeated vertex in cell " + std::to_string(c), c);
    }
    throw_code(FB_ERR_INVALID_ARGUMENT, "cell vertex index out of range in cell " + std::to_string(c), c);
  }
  A.home = dev;
  A.dev.emplace(dev, p);  // owned from here on (freed by ~fb_assembly)
  A.total_nbr = P.total_nbr;
  if (bad[2] >= 0)
    throw_code(FB_ERR_INVALID_ARGUMENT, "vertex degree exceeds 255 at vertex " + std::to_string(bad[2]), -1);
  if (A.total_nbr * A.nc > INT32_MAX || A.rows() > INT32_MAX)
    throw_code(FB_ERR_INVALID_ARGUMENT, "assembled operator exceeds 32-bit column indices", -1);
}

template <class T>
T* upload(const std::vector<T>& h)
{
  T* d = nullptr;
  cuda_check(cudaMalloc(&d, std::max<size_t>(h.size(), 1) * sizeof(T)), "cudaMalloc");
  if (!h.empty())
    cuda_check(cudaMemcpy(d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice), "cudaMemcpy plan");
  return d;
}

template <class T>
void download(std::vector<T>& h, const T* d, int64_t n)
{
  h.resize(n);
  if (n > 0)
    cuda_check(cudaMemcpy(h.data(), d, n * sizeof(T), cudaMemcpyDeviceToHost), "cudaMemcpy plan");
}

// Host copies of a device-built plan (for the pattern, or another device).
// Caller holds A.mu.
void ensure_host(const fb_assembly& A)
{
  if (A.home < 0 || !A.nbr_ptr.empty())
    return;
  auto& M = const_cast<fb_assembly&>(A);
  const DevPlan& p = A.dev.at(A.home);
  int cur = 0;
  cuda_check(cudaGetDevice(&cur), "cudaGetDevice");
  cuda_check(cudaSetDevice(A.home), "cudaSetDevice");
  const int64_t ngroups = (A.nv + 31) / 32;
  download(M.goff, p.goff, ngroups + 1);
  download(M.spk, p.spk, M.goff.back());
  download(M.spos, p.spos, M.goff.back());
  download(M.nbr, p.nbr, A.total_nbr);
  download(M.nbr_ptr, p.nbr_ptr, A.nv + 1);
  cuda_check(cudaSetDevice(cur), "cudaSetDevice");
}

const DevPlan& plan_on(const fb_assembly& A, int dev)
{
  std::lock_guard<std::mutex> lock(A.mu);
  auto it = A.dev.find(dev);
  if (it != A.dev.end())
    return it->second;
  ensure_host(A);
  DevPlan p;
  p.goff = upload(A.goff);
  p.spk = upload(A.spk);
  p.spos = upload(A.spos);
  p.nbr_ptr = upload(A.nbr_ptr);
  return A.dev.emplace(dev, p).first->second;
}

void check_pair(const fb_assembly* a, const fb_variant* v, int64_t store_len, int64_t nnz)
{
  if (!a)
    invalid("null assembly plan");
  if (!v)
    invalid("null kernel variant");
  if (v->dim != a->dim)
    invalid("assembly plan and variant differ in dimension");
  if ((v->op == FB_ELASTICITY) != (a->op == FB_ELASTICITY))
    invalid("assembly plan and variant differ in operator shape");
  if (store_len < a->ne * v->krows * v->krows)
    invalid("element matrix store shorter than num_elements * krows^2");
  if (nnz != a->nnz())
    invalid("values length must equal the plan's nnz");
}

void check_flags(int flags)
{
  if (flags & ~(FB_ASSEMBLE_SYMMETRIC | FB_ASSEMBLE_BLOCK_DIAGONAL))
    invalid("unknown assembly flags");
}

void launch_on(const fb_assembly& A, const fb_variant& v, const void* store, void* values, int flags, int dev,
               cudaStream_t st)
{
  const DevPlan& p = plan_on(A, dev);
  fbk::AsmArgs g;
  g.goff = p.goff;
  g.spk = p.spk;
  g.spos = p.spos;
  g.nbr_ptr = p.nbr_ptr;
  g.store = store;
  g.values = values;
  g.nv = A.nv;
  // column reads need the caller's symmetry promise and 16-byte alignment
  g.sym = (flags & FB_ASSEMBLE_SYMMETRIC) && (reinterpret_cast<uintptr_t>(store) & 15u) == 0 ? 1 : 0;
  g.diag = (flags & FB_ASSEMBLE_BLOCK_DIAGONAL) && A.nc > 1 ? 1 : 0;
  cuda_check(fbk::launch_assemble(A.dim, A.nc, v.cfg.precision, g, st), "assemble kernel launch");
}

void check_packed(const fb_assembly* a, const fb_variant* v, const void* g, int64_t g_len, const double* coeffs,
                  int64_t coeffs_len, const void* values, int64_t nnz)
{
  check_pair(a, v, a ? a->ne * (v ? v->krows * v->krows : 0) : 0, nnz);
  const int64_t dd = static_cast<int64_t>(a->dim) * a->dim;
  if (v->path == fbk::kDense)
    invalid("packed-geometry assembly needs a K with the P1 sparsity pattern");
  if (a->ne > 0 && !g)
    invalid("null packed geometry");
  if (g_len < a->ne * dd)
    invalid("packed geometry shorter than num_elements * dim^2");
  if (reinterpret_cast<uintptr_t>(g) % scalar_size(v->cfg.precision) != 0)
    invalid("packed geometry is not aligned to its scalar size");
  if (v->op == FB_WEIGHTED_LAPLACIAN)
  {
    if (a->ne > 0 && !coeffs)
      invalid("weighted Laplacian needs nodal coefficients");
    if (coeffs_len < a->ne * (a->dim + 1))
      invalid("coefficients shorter than num_elements * (dim+1)");
  }
  if (a->nnz() > 0 && !values)
    invalid("null values buffer");
}

void launch_packed_on(const fb_assembly& A, const fb_variant& v, const void* g, const double* coeffs, void* values,
                      int dev, cudaStream_t st)
{
  const DevPlan& p = plan_on(A, dev);
  fbk::AsmArgs ga;
  ga.goff = p.goff;
  ga.spk = p.spk;
  ga.spos = p.spos;
  ga.nbr_ptr = p.nbr_ptr;
  ga.values = values;
  ga.nv = A.nv;
  // vector loads need a 16-byte aligned G; else the kernel reads it scalar-wise
  ga.g_in = g;
  ga.g_len = (reinterpret_cast<uintptr_t>(g) & 15u) == 0 ? A.ne * A.dim * A.dim : -1;
  ga.coeffs = v.op == FB_WEIGHTED_LAPLACIAN ? coeffs : nullptr;
  fbk::LaunchSpec s;
  s.op = v.op;
  s.dim = v.dim;
  s.prec = v.cfg.precision;
  s.mode = v.cfg.mode;
  s.path = v.path;
  s.from_g = 1;
  cuda_check(fbk::launch_assemble_g(s, ga, v.kp, st), "packed assembly kernel launch");
}

}  // namespace

extern "C" {

fb_assembly* fb_assembly_create(int op, int dim, const int32_t* cells, int64_t ne, int64_t nv, fb_error* err)
{
  std::unique_ptr<fb_assembly> A;
  const int rc = guarded(err,
                         [&]
                         {
                           if (dim != 2 && dim != 3)
                             invalid("unsupported spatial dimension " + std::to_string(dim));
                           if (op < FB_LAPLACIAN || op > FB_WEIGHTED_LAPLACIAN)
                             invalid("unknown operator");
                           if (ne < 0 || nv < 0 || nv > INT32_MAX || ne >= (int64_t(1) << 30))
                             invalid("mesh sizes out of range for assembly");
                           if (ne > 0 && !cells)
                             invalid("null cells");
                           auto fresh = [&]
                           {
                             A = std::make_unique<fb_assembly>();
                             A->op = op;
                             A->dim = dim;
                             A->nb = dim + 1;
                             A->nc = op == FB_ELASTICITY ? dim : 1;
                             A->nv = nv;
                             A->ne = ne;
                           };
                           fresh();
                           const int cdev = ne > 0 ? pointer_device(cells) : -1;
                           if (cdev >= 0)
                             build_plan_gpu(*A, cells, cdev);  // device-resident connectivity
                           else if (ne >= kGpuPlanMinElements && device_count() > 0 && !std::getenv("FB_PLAN_HOST"))
                           {
                             // host connectivity of a large mesh: upload it and
                             // build on the current GPU (same plan array for
                             // array; 16.8 M tets: ~25 ms vs ~1 s on the host).
                             // A CUDA failure there (out of memory, a device
                             // in exclusive use) falls back to the host builder;
                             // invalid input still fails as invalid input.
                             bool gpu_ok = false;
                             try
                             {
                               int dev = 0;
                               cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
                               const size_t bytes = static_cast<size_t>(ne) * (dim + 1) * sizeof(int32_t);
                               int32_t* d = nullptr;
                               cuda_check(cudaMalloc(&d, bytes), "cudaMalloc");
                               try
                               {
                                 cuda_check(cudaMemcpy(d, cells, bytes, cudaMemcpyHostToDevice), "upload cells");
                                 build_plan_gpu(*A, d, dev);
                               }
                               catch (...)
                               {
                                 cudaFree(d);
                                 throw;
                               }
                               cudaFree(d);
                               gpu_ok = true;
                             }
                             catch (const Error& e)
                             {
                               if (e.code != FB_ERR_CUDA)
                                 throw;
                               cudaGetLastError();  // clear the sticky-free error state
                             }
                             if (!gpu_ok)
                             {
                               fresh();
                               build_plan(*A, cells);
                             }
                           }
                           else
                             build_plan(*A, cells);
                         });
  return rc == FB_OK ? A.release() : nullptr;
}

void fb_assembly_free(fb_assembly* a) { delete a; }
int64_t fb_assembly_rows(const fb_assembly* a) { return a ? a->rows() : -1; }
int64_t fb_assembly_nnz(const fb_assembly* a) { return a ? a->nnz() : -1; }

int fb_assembly_pattern(const fb_assembly* a, int64_t* row_ptr, int64_t row_ptr_len, int32_t* col_idx,
                        int64_t nnz, fb_error* err)
{
  return guarded(err,
                 [&]
                 {
                   if (!a)
                     invalid("null assembly plan");
                   if (row_ptr_len != a->rows() + 1 || nnz != a->nnz())
                     invalid("pattern buffers must hold rows+1 offsets and nnz columns");
                   {
                     std::lock_guard<std::mutex> lock(a->mu);
                     ensure_host(*a);
                   }
                   const int nc = a->nc;
                   int64_t z = 0;
                   row_ptr[0] = 0;
                   for (int64_t v = 0; v < a->nv; ++v)
                     for (int ci = 0; ci < nc; ++ci)
                     {
                       for (int64_t k = a->nbr_ptr[v]; k < a->nbr_ptr[v + 1]; ++k)
                         for (int cj = 0; cj < nc; ++cj)
                           col_idx[z++] = static_cast<int32_t>(a->nbr[k] * nc + cj);
                       row_ptr[v * nc + ci + 1] = z;
                     }
                 });
}

int fb_assemble_async(const fb_assembly* a, const fb_variant* v, const void* store, int64_t store_len,
                      void* values, int64_t nnz, int flags, void* stream, fb_error* err)
{
  return guarded(err,
                 [&]
                 {
                   check_pair(a, v, store_len, nnz);
                   check_flags(flags);
                   int dev = 0;
                   cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
                   launch_on(*a, *v, store, values, flags, dev, static_cast<cudaStream_t>(stream));
                 });
}

int fb_assemble_packed_async(const fb_assembly* a, const fb_variant* v, const void* g, int64_t g_len,
                             const double* coeffs, int64_t coeffs_len, void* values, int64_t nnz, void* stream,
                             fb_error* err)
{
  return guarded(err,
                 [&]
                 {
                   check_packed(a, v, g, g_len, coeffs, coeffs_len, values, nnz);
                   int dev = 0;
                   cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
                   launch_packed_on(*a, *v, g, coeffs, values, dev, static_cast<cudaStream_t>(stream));
                 });
}

int fb_assemble_packed(const fb_assembly* a, const fb_variant* v, const void* g, int64_t g_len,
                       const double* coeffs, int64_t coeffs_len, void* values, int64_t nnz, int device,
                       fb_error* err)
{
  return guarded(err,
                 [&]
                 {
                   check_packed(a, v, g, g_len, coeffs, coeffs_len, values, nnz);
                   if (device_count() == 0)
                     throw_code(FB_ERR_NO_DEVICE, "no CUDA device available");
                   const int gdev = pointer_device(g), vdev = pointer_device(values);
                   const int dev = gdev >= 0 ? gdev : (vdev >= 0 ? vdev : std::max(device, 0));
                   const bool weighted = v->op == FB_WEIGHTED_LAPLACIAN;
                   const int cdev = weighted ? pointer_device(coeffs) : dev;
                   int cur = 0;
                   cuda_check(cudaGetDevice(&cur), "cudaGetDevice");
                   cuda_check(cudaSetDevice(dev), "cudaSetDevice");
                   const size_t ss = scalar_size(v->cfg.precision);
                   const size_t gbytes = static_cast<size_t>(a->ne) * a->dim * a->dim * ss;
                   const size_t cbytes = static_cast<size_t>(a->ne) * (a->dim + 1) * sizeof(double);
                   const size_t vbytes = static_cast<size_t>(nnz) * ss;
                   std::vector<void*> tmp;
                   cudaStream_t st = nullptr;
                   auto stage_in = [&](const void* src, size_t bytes) -> void*
                   {
                     void* d = nullptr;
                     cuda_check(cudaMalloc(&d, std::max<size_t>(bytes, 16)), "cudaMalloc");
                     tmp.push_back(d);
                     if (bytes)
                       cuda_check(cudaMemcpyAsync(d, src, bytes, cudaMemcpyDefault, st), "upload");
                     return d;
                   };
                   auto cleanup = [&]
                   {
                     if (st)
                       cudaStreamSynchronize(st);
                     for (void* p : tmp)
                       cudaFree(p);
                     if (st)
                       cudaStreamDestroy(st);
                     cudaSetDevice(cur);
                   };
                   try
                   {
                     cuda_check(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "cudaStreamCreate");
                     const void* dg = gdev == dev ? g : stage_in(g, gbytes);
                     const double* dc =
                         !weighted || cdev == dev ? coeffs : static_cast<const double*>(stage_in(coeffs, cbytes));
                     void* dv = values;
                     if (vdev != dev)
                     {
                       cuda_check(cudaMalloc(&dv, std::max<size_t>(vbytes, 16)), "cudaMalloc");
                       tmp.push_back(dv);
                     }
                     launch_packed_on(*a, *v, dg, dc, dv, dev, st);
                     if (vdev != dev && vbytes)
                       cuda_check(cudaMemcpyAsync(values, dv, vbytes, cudaMemcpyDefault, st), "download values");
                     cuda_check(cudaStreamSynchronize(st), "cudaStreamSynchronize");
                   }
                   catch (...)
                   {
                     cleanup();
                     throw;
                   }
                   cleanup();
                 });
}

int fb_assemble(const fb_assembly* a, const fb_variant* v, const void* store, int64_t store_len, void* values,
                int64_t nnz, int flags, int device, fb_error* err)
{
  return guarded(err,
                 [&]
                 {
                   check_pair(a, v, store_len, nnz);
                   check_flags(flags);
                   if (device_count() == 0)
                     throw_code(FB_ERR_NO_DEVICE, "no CUDA device available");
                   const int sdev = pointer_device(store), vdev = pointer_device(values);
                   const int dev = sdev >= 0 ? sdev : (vdev >= 0 ? vdev : std::max(device, 0));
                   int cur = 0;
                   cuda_check(cudaGetDevice(&cur), "cudaGetDevice");
                   cuda_check(cudaSetDevice(dev), "cudaSetDevice");
                   const size_t ss = scalar_size(v->cfg.precision);
                   const size_t sbytes = static_cast<size_t>(a->ne) * v->krows * v->krows * ss;
                   const size_t vbytes = static_cast<size_t>(nnz) * ss;
                   void* ds = const_cast<void*>(store);
                   void* dv = values;
                   void* tmp_s = nullptr;
                   void* tmp_v = nullptr;
                   cudaStream_t st = nullptr;
                   try
                   {
                     cuda_check(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "cudaStreamCreate");
                     if (sdev != dev)
                     {
                       cuda_check(cudaMalloc(&tmp_s, std::max<size_t>(sbytes, 16)), "cudaMalloc");
                       cuda_check(cudaMemcpyAsync(tmp_s, store, sbytes, cudaMemcpyDefault, st), "upload store");
                       ds = tmp_s;
                     }
                     if (vdev != dev)
                     {
                       cuda_check(cudaMalloc(&tmp_v, std::max<size_t>(vbytes, 16)), "cudaMalloc");
                       dv = tmp_v;
                     }
                     launch_on(*a, *v, ds, dv, flags, dev, st);
                     if (tmp_v)
                       cuda_check(cudaMemcpyAsync(values, tmp_v, vbytes, cudaMemcpyDefault, st), "download values");
                     cuda_check(cudaStreamSynchronize(st), "cudaStreamSynchronize");
                   }
                   catch (...)
                   {
                     if (st)
                       cudaStreamSynchronize(st);
                     cudaFree(tmp_s);
                     cudaFree(tmp_v);
                     if (st)
                       cudaStreamDestroy(st);
                     cudaSetDevice(cur);
                     throw;
                   }
                   cudaFree(tmp_s);
                   cudaFree(tmp_v);
                   cudaStreamDestroy(st);
                   cudaSetDevice(cur);
                 });
}

}  // extern "C"
