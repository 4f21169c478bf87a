// fb_capi.cpp -- the extern "C" boundary (include/fembatch_b200.h).
//
// Responsibilities: argument validation with the reference's exception texts
// (src/engine.cpp:301-376, src/kernel_config.cpp:43-55), K structure
// validation and kernel-path choice at specialize time, per-device workspace
// and streams, host<->device staging with a two-stream chunk pipeline,
// element-range sharding across devices (one host thread per device, no
// collectives), and mapping the kernel's status words back to the
// reference's degenerate-cell error.
#include <algorithm>
#include <array>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <limits>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/fembatch_b200.h"
#include "fb_capi_util.h"
#include "fb_devcache.h"
#include "fb_host.h"
#include "fb_internal.h"

namespace fbk {
std::atomic<long long>& launch_counter();
}

namespace {

using namespace fbc;

constexpr long long kStatusInit = 0x7f7f7f7f7f7f7f7fLL;  // memset(0x7f) pattern

// ----------------------------------------------------- config validation
// src/kernel_config.cpp:43-55
void validate_config(const fb_kernel_config& c)
{
  if (c.element_batch_size < 1)
    invalid("element_batch_size must be positive");
  if (c.num_concurrent_elements < 1)
    invalid("num_concurrent_elements must be positive");
  if (c.element_batch_size % c.num_concurrent_elements != 0)
    invalid("num_concurrent_elements (" + std::to_string(c.num_concurrent_elements)
            + ") must divide element_batch_size (" + std::to_string(c.element_batch_size) + ")");
  if (c.precision != FB_F32 && c.precision != FB_F64)
    invalid("unknown precision");
  if (c.mode != FB_STRICT && c.mode != FB_FAST)
    invalid("unknown arithmetic mode");
  if (c.store < FB_STORE_AUTO || c.store > FB_STORE_TMA)
    invalid("unknown store strategy");
}

int64_t store_len(int krows, int64_t ne, int bs)
{
  const int64_t nbatch = (ne + bs - 1) / bs;
  return nbatch * bs * static_cast<int64_t>(krows) * krows;
}


// ------------------------------------------------- K structure analysis
template <class S>
void analyse_k(fb_variant& v)
{
  const int nb = v.nb, kr = v.krows, nc = v.ncoef, dim = v.dim, dd = dim * dim;
  auto K = [&](int i, int j, int c, int t)
  { return static_cast<S>(v.k[static_cast<size_t>((static_cast<int64_t>(i + j * kr) * nc + c) * dd + t)]); };

  bool pattern = true, sym = true;
  for (int i = 0; i < kr; ++i)
    for (int j = 0; j < kr; ++j)
      for (int c = 0; c < nc; ++c)
        for (int t = 0; t < dd; ++t)
        {
          const S val = K(i, j, c, t);
          if (val != val)  // NaN: only the dense path reproduces its propagation
            pattern = false;
          const int a = i % nb, ci = i / nb, b = j % nb, cj = j / nb;
          const int mu = t / dim, nu = t % dim;
          if (ci != cj)
          {
            if (val != S(0))
              pattern = false;
            continue;
          }
          const bool nz = (a == 0 || mu == a - 1) && (b == 0 || nu == b - 1);
          if (!nz && val != S(0))
            pattern = false;
          if (ci > 0 && !(val == K(a, b, c, t)))  // elasticity: equal component blocks
            pattern = false;
          if (ci == 0 && !(val == K(b, a, c, nu * dim + mu)))
            sym = false;
        }
  // uniform magnitude: K = sigma_ab * kappa_c on the P1 pattern, sigma_ab = -1
  // iff exactly one of a, b is 0 (reference gradients), kappa_c > 0 finite
  bool uniform = pattern && sym;
  std::vector<S> kappa(nc);
  for (int c = 0; c < nc && uniform; ++c)
  {
    kappa[c] = K(0, 0, c, 0);
    if (!(kappa[c] > S(0)) || !(kappa[c] < std::numeric_limits<S>::infinity()))
      uniform = false;
    for (int a = 0; a < nb && uniform; ++a)
      for (int b = 0; b < nb && uniform; ++b)
        for (int t = 0; t < dd; ++t)
        {
          const int mu = t / dim, nu = t % dim;
          if (!((a == 0 || mu == a - 1) && (b == 0 || nu == b - 1)))
            continue;
          const S want = ((a == 0) != (b == 0)) ? -kappa[c] : kappa[c];
          if (!(K(a, b, c, t) == want))
            uniform = false;
        }
  }
  v.path = !pattern ? fbk::kDense : (uniform ? fbk::kUniformSym : (sym ? fbk::kSparseSym : fbk::kSparse));

  static_assert(sizeof(fbk::KParamBlob) >= 16 * 4 * 9 * sizeof(double), "blob too small");
  S* kp = reinterpret_cast<S*>(v.kp.bytes);
  if (uniform)
    for (int c = 0; c < nc; ++c)
      kp[c] = kappa[c];
  else
    for (int a = 0; a < nb; ++a)
      for (int b = 0; b < nb; ++b)
        for (int c = 0; c < nc; ++c)
          for (int t = 0; t < dd; ++t)
            kp[((a * nb + b) * nc + c) * dd + t] = K(a, b, c, t);

  v.kdense.resize(v.k.size() * sizeof(S));
  S* kd = reinterpret_cast<S*>(v.kdense.data());
  for (size_t t = 0; t < v.k.size(); ++t)
    kd[t] = static_cast<S>(v.k[t]);
}

// ------------------------------------------------------ device contexts
struct Buf {
  void* p = nullptr;
  size_t n = 0;
  void release()
  {
    if (p)
      cudaFree(p);
    p = nullptr;
    n = 0;
  }
  void* get(size_t need)
  {
    if (need > n)
    {
      if (p)
        cudaFree(p);
      p = nullptr;
      n = 0;
      cuda_check(cudaMalloc(&p, std::max<size_t>(need, 256)), "cudaMalloc");
      n = std::max<size_t>(need, 256);
    }
    return p;
  }
};

struct DeviceCtx {
  std::mutex mu;
  bool ready = false;
  cudaStream_t st[2] = {nullptr, nullptr};
  cudaEvent_t ev = nullptr;
  Buf vtx, coeff_all, status;
  Buf in[2], coeff[2], out[2];
  long long* status_host = nullptr;
  void init(int dev)
  {
    if (ready)
      return;
    cuda_check(cudaSetDevice(dev), "cudaSetDevice");
    for (auto& s : st)
      cuda_check(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "cudaStreamCreate");
    cuda_check(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "cudaEventCreate");
    cuda_check(cudaMallocHost(&status_host, 2 * sizeof(long long)), "cudaMallocHost");
    ready = true;
  }
  // caller holds mu and has made the device current
  void release()
  {
    if (!ready)
      return;
    for (auto& s : st)
      cudaStreamDestroy(s);
    cudaEventDestroy(ev);
    cudaFreeHost(status_host);
    for (Buf* b : {&vtx, &coeff_all, &status, &in[0], &in[1], &coeff[0], &coeff[1], &out[0], &out[1]})
      b->release();
    st[0] = st[1] = nullptr;
    ev = nullptr;
    status_host = nullptr;
    ready = false;
  }
};

// Restores the calling thread's current device on every exit path: the
// blocking entry points switch devices internally (run_on_device) and must
// not leave the caller on another GPU.
struct DeviceGuard {
  int dev = -1;
  DeviceGuard() { cudaGetDevice(&dev); }
  ~DeviceGuard()
  {
    if (dev >= 0)
      cudaSetDevice(dev);
  }
};

std::mutex g_ctx_mu;
std::map<int, std::unique_ptr<DeviceCtx>>& contexts()
{
  static std::map<int, std::unique_ptr<DeviceCtx>> m;
  return m;
}

DeviceCtx& ctx_for(int dev)
{
  std::lock_guard<std::mutex> lock(g_ctx_mu);
  auto& m = contexts();
  auto it = m.find(dev);
  if (it == m.end())
    it = m.emplace(dev, std::make_unique<DeviceCtx>()).first;
  return *it->second;
}

const void* kdense_on(const fb_variant& v, int dev)
{
  if (v.path != fbk::kDense)
    return nullptr;
  std::lock_guard<std::mutex> lock(v.mu);
  auto it = v.kdense_dev.find(dev);
  if (it != v.kdense_dev.end())
    return it->second;
  void* p = nullptr;
  cuda_check(cudaMalloc(&p, v.kdense.size()), "cudaMalloc");
  cuda_check(cudaMemcpy(p, v.kdense.data(), v.kdense.size(), cudaMemcpyHostToDevice), "cudaMemcpy K");
  v.kdense_dev[dev] = p;
  return p;
}

[[noreturn]] void raise_status(long long degenerate, long long bad_index)
{
  // The reference reports the first failing cell in slot order
  // (geometry.cpp:280-282 via pack_geometry's serial loop).
  if (bad_index < degenerate)
    throw_code(FB_ERR_INVALID_ARGUMENT,
               "cell vertex index out of range in cell " + std::to_string(bad_index), bad_index);
  throw_code(FB_ERR_RUNTIME, "degenerate element: det(J) <= 0 in cell " + std::to_string(degenerate),
             degenerate);
}

void check_status_words(const long long* w)
{
  if (w[0] != kStatusInit || w[1] != kStatusInit)
    raise_status(w[0], w[1]);
}

// ------------------------------------------------------------ the job
enum class Kind { Mesh, Packed, Pack };

struct Job {
  Kind kind = Kind::Mesh;
  const fb_variant* var = nullptr;  // null for Pack
  int dim = 2, prec = 1, nb = 3, nk = 9;  // nk: output scalars per slot
  int64_t nv = 0, ne = 0, nslots = 0;
  const double* vtx = nullptr;
  const int32_t* cells = nullptr;
  const double* coeffs = nullptr;
  const void* g = nullptr;
  void* out = nullptr;
  int vtx_dev = -1, cells_dev = -1, coeff_dev = -1, g_dev = -1, out_dev = -1;
  fbk::LaunchSpec spec{};
};

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// Elements whose connectivity / coefficients slots [s0, s1) touch.
void element_window(const Job& j, int64_t s0, int64_t s1, int64_t& lo, int64_t& hi)
{
  lo = std::min(s0, j.ne - 1);
  hi = std::min(std::max(s1, lo + 1), j.ne);
}

// Kernels index slots with 32-bit locals: split launches at 2^30 slots.
// FB_TEST_MAX_LAUNCH_SLOTS (environment, test hook) lowers the split so the
// multi-launch path is exercised at small sizes.
const int64_t kMaxLaunchSlots = []
{
  const char* e = std::getenv("FB_TEST_MAX_LAUNCH_SLOTS");
  const long long v = e ? std::atoll(e) : 0;
  return v >= 32 && v < (1ll << 30) ? static_cast<int64_t>(v / 32 * 32) : int64_t(1) << 30;
}();

void launch_integrate_chunked(const fbk::LaunchSpec& spec, const fbk::LaunchArgs& a, const fbk::KParamBlob& kp,
                              int nk, int dd, size_t ss, cudaStream_t st)
{
  for (int64_t off = 0; off < a.nloc; off += kMaxLaunchSlots)
  {
    fbk::LaunchArgs c = a;
    c.slot0 = a.slot0 + off;
    c.nloc = std::min(kMaxLaunchSlots, a.nloc - off);
    c.out = static_cast<char*>(a.out) + off * nk * ss;
    if (a.g_in)
      c.g_in = static_cast<const char*>(a.g_in) + off * dd * ss;
    cuda_check(fbk::launch_integrate(spec, c, kp, st), "integrate kernel launch");
  }
}

// pack_geometry: the same 2^30-slot split (32-bit local slot indices)
void launch_pack_chunked(int dim, int prec, const fbk::LaunchArgs& a, cudaStream_t st)
{
  const int64_t dd = static_cast<int64_t>(dim) * dim;
  for (int64_t off = 0; off < a.nloc; off += kMaxLaunchSlots)
  {
    fbk::LaunchArgs c = a;
    c.slot0 = a.slot0 + off;
    c.nloc = std::min(kMaxLaunchSlots, a.nloc - off);
    c.out = static_cast<char*>(a.out) + off * dd * scalar_size(prec);
    cuda_check(fbk::launch_pack(dim, prec, c, st), "pack kernel launch");
  }
}

void launch(const Job& j, const fbk::LaunchArgs& a, cudaStream_t st)
{
  if (j.kind == Kind::Pack)
    launch_pack_chunked(j.dim, j.prec, a, st);
  else
    launch_integrate_chunked(j.spec, a, j.var->kp, j.nk, j.dim * j.dim, scalar_size(j.prec), st);
}

// Contiguous tile-aligned slot shards of a device list: outputs
// concatenate.  Exported as fb_shard_bounds.
std::vector<int64_t> shard_bounds(int64_t nslots, int parts)
{
  if (parts < 1)
    invalid("worker count must be >= 1");
  if (nslots < 0)
    invalid("negative slot count");
  const int64_t tiles = fbk::num_tiles(nslots);
  std::vector<int64_t> bound(parts + 1);
  for (int g = 0; g <= parts; ++g)
    bound[g] = std::min(nslots, tiles * g / parts * fbk::kTile);
  return bound;
}

// Runs slots [s0, s1) of the job on device `dev`.  Host buffers are staged in
// chunks through double-buffered device workspace on two streams, so chunk
// i's device->host copy overlaps chunk i+1's upload and kernel.
void run_on_device(const Job& j, int dev, int64_t s0, int64_t s1, long long* status_out)
{
  DeviceCtx& ctx = ctx_for(dev);
  std::lock_guard<std::mutex> lock(ctx.mu);
  ctx.init(dev);
  cuda_check(cudaSetDevice(dev), "cudaSetDevice");
  const size_t ss = scalar_size(j.prec);
  const int nb = j.nb;
  const int dd = j.dim * j.dim;

  fbk::LaunchArgs base{};
  base.nv = j.nv;
  base.ne = j.ne;
  base.kdense = j.var ? kdense_on(*j.var, dev) : nullptr;

  long long* status = static_cast<long long*>(ctx.status.get(2 * sizeof(long long)));
  cuda_check(cudaMemsetAsync(status, 0x7f, 2 * sizeof(long long), ctx.st[0]), "cudaMemsetAsync");
  base.status = status;

  if (j.kind != Kind::Packed && j.nv > 0)
  {
    if (j.vtx_dev == dev)
      base.vtx = j.vtx;
    else
    {
      double* d = static_cast<double*>(ctx.vtx.get(j.nv * j.dim * sizeof(double)));
      cuda_check(cudaMemcpyAsync(d, j.vtx, j.nv * j.dim * sizeof(double), cudaMemcpyDefault,
                                 ctx.st[0]),
                 "upload vertices");
      base.vtx = d;
    }
  }
  base.vtx_aligned16 = aligned16(base.vtx);
  cuda_check(cudaEventRecord(ctx.ev, ctx.st[0]), "cudaEventRecord");
  cuda_check(cudaStreamWaitEvent(ctx.st[1], ctx.ev, 0), "cudaStreamWaitEvent");

  const bool direct_out = j.out_dev == dev;
  const bool whole = direct_out && (j.kind == Kind::Packed ? j.g_dev == dev : j.cells_dev == dev)
                     && (j.coeffs == nullptr || j.coeff_dev == dev);
  // Host-staged jobs run as a chunk pipeline whose outputs start at ~4 MB and
  // double up to 64 MB: the first device->host copy starts early (PCIe D2H of
  // the store dominates), later chunks amortise per-launch cost.  A fully
  // device-resident job is one chunk.
  auto slots_for = [&](int64_t bytes)
  {
    const int64_t per = std::max<int64_t>(1, bytes / (j.nk * static_cast<int64_t>(ss)));
    return std::max<int64_t>(fbk::kTile, per / fbk::kTile * fbk::kTile);
  };
  int64_t chunk = whole ? s1 - s0 : slots_for(4ll << 20);
  const int64_t chunk_max = whole ? s1 - s0 : slots_for(64ll << 20);

  int which = 0;
  for (int64_t c0 = s0, c1 = 0; c0 < s1; c0 = c1, which ^= 1, chunk = std::min(chunk_max, 2 * chunk))
  {
    c1 = std::min(s1, c0 + chunk);
    cudaStream_t st = ctx.st[which];
    fbk::LaunchArgs a = base;
    a.slot0 = c0;
    a.nloc = c1 - c0;
    int64_t lo = 0, hi = 0;
    if (j.ne > 0)
      element_window(j, c0, c1, lo, hi);

    if (j.kind == Kind::Packed)
    {
      if (j.g_dev == dev)
        a.g_in = static_cast<const char*>(j.g) + c0 * dd * ss;
      else
      {
        void* d = ctx.in[which].get((c1 - c0) * dd * ss);
        cuda_check(cudaMemcpyAsync(d, static_cast<const char*>(j.g) + c0 * dd * ss, (c1 - c0) * dd * ss,
                                   cudaMemcpyDefault, st),
                   "upload G");
        a.g_in = d;
      }
    }
    else if (j.ne > 0)
    {
      if (j.cells_dev == dev)
        a.cells = j.cells;
      else
      {
        int32_t* d = static_cast<int32_t*>(ctx.in[which].get((hi - lo) * nb * sizeof(int32_t)));
        cuda_check(cudaMemcpyAsync(d, j.cells + lo * nb, (hi - lo) * nb * sizeof(int32_t),
                                   cudaMemcpyDefault, st),
                   "upload cells");
        a.cells = d - lo * nb;
      }
    }
    a.cells_aligned16 = aligned16(a.cells);
    if (j.coeffs)
    {
      if (j.coeff_dev == dev)
        a.coeffs = j.coeffs;
      else
      {
        double* d = static_cast<double*>(ctx.coeff[which].get((hi - lo) * nb * sizeof(double)));
        cuda_check(cudaMemcpyAsync(d, j.coeffs + lo * nb, (hi - lo) * nb * sizeof(double),
                                   cudaMemcpyDefault, st),
                   "upload coefficients");
        a.coeffs = d - lo * nb;
      }
    }
    const size_t out_bytes = (c1 - c0) * j.nk * ss;
    void* dout = direct_out ? static_cast<char*>(j.out) + c0 * j.nk * ss : ctx.out[which].get(out_bytes);
    a.out = dout;
    fbk::LaunchSpec spec = j.spec;
    if (j.kind != Kind::Pack && !aligned16(dout))
      spec.staged = 0;
    Job jj = j;
    jj.spec = spec;
    launch(jj, a, st);
    if (!direct_out)
      cuda_check(cudaMemcpyAsync(static_cast<char*>(j.out) + c0 * j.nk * ss, dout, out_bytes,
                                 cudaMemcpyDefault, st),
                 "download store");
  }
  cuda_check(cudaEventRecord(ctx.ev, ctx.st[1]), "cudaEventRecord");
  cuda_check(cudaStreamWaitEvent(ctx.st[0], ctx.ev, 0), "cudaStreamWaitEvent");
  cuda_check(cudaMemcpyAsync(ctx.status_host, status, 2 * sizeof(long long), cudaMemcpyDeviceToHost,
                             ctx.st[0]),
             "download status");
  cuda_check(cudaStreamSynchronize(ctx.st[0]), "cudaStreamSynchronize");
  status_out[0] = ctx.status_host[0];
  status_out[1] = ctx.status_host[1];
}

void run_job(const Job& j, const int* devices, int ndev)
{
  DeviceGuard keep_device;  // the caller's current device survives the call
  const int have = device_count();
  if (have == 0)
    throw_code(FB_ERR_NO_DEVICE, "no CUDA device available");
  std::vector<int> devs;
  if (devices && ndev > 0)
    devs.assign(devices, devices + ndev);
  else
  {
    int pick = 0;
    for (int d : {j.out_dev, j.cells_dev, j.g_dev, j.vtx_dev})
      if (d >= 0)
      {
        pick = d;
        break;
      }
    devs.push_back(pick);
  }
  for (int d : devs)
    if (d < 0 || d >= have)
      invalid("device " + std::to_string(d) + " does not exist");
  // Operands may live on the host or on any device: each shard device works
  // on its own slice and the staging copies use cudaMemcpyDefault, so a
  // device-resident operand on another GPU moves over NVLink peer copies
  // (e.g. every GPU's output slice gathered into one device's store).
  if (j.nslots == 0)
    return;

  // contiguous tile-aligned slot shards: outputs concatenate
  const int P = static_cast<int>(devs.size());
  const std::vector<int64_t> bound = shard_bounds(j.nslots, P);
  std::vector<std::array<long long, 2>> st(P, {kStatusInit, kStatusInit});
  std::vector<std::exception_ptr> errs(P);
  auto body = [&](int g)
  {
    try
    {
      if (bound[g + 1] > bound[g])
        run_on_device(j, devs[g], bound[g], bound[g + 1], st[g].data());
    }
    catch (...)
    {
      errs[g] = std::current_exception();
    }
  };
  if (P == 1)
    body(0);
  else
  {
    std::vector<std::thread> pool;
    for (int g = 0; g < P; ++g)
      pool.emplace_back(body, g);
    for (auto& t : pool)
      t.join();
  }
  for (auto& e : errs)
    if (e)
      std::rethrow_exception(e);
  long long w[2] = {kStatusInit, kStatusInit};
  for (auto& s : st)
  {
    w[0] = std::min(w[0], s[0]);
    w[1] = std::min(w[1], s[1]);
  }
  check_status_words(w);
}

const fb_variant& checked(const fb_variant* v)
{
  if (!v)
    invalid("null kernel variant");
  return *v;
}

// src/engine.cpp:346-371
void validate_coefficients(const fb_variant& v, int64_t ne, const double* coeffs)
{
  if (v.op == FB_WEIGHTED_LAPLACIAN)
  {
    if (!coeffs)
      invalid("form requires a coefficient field");
    if (ne == 0)
      invalid("cannot integrate a coefficient form over zero elements");
  }
  else if (coeffs)
    invalid("form takes no coefficient field");
}

void validate_out(const fb_variant& v, int64_t nslots, void* out, int64_t out_len)
{
  const int64_t want = nslots * v.krows * v.krows;
  if (out_len != want)
    invalid("output buffer holds " + std::to_string(out_len) + " scalars; the store needs "
            + std::to_string(want));
  if (want > 0 && !out)
    invalid("null output buffer");
}

void validate_mesh_view(const fb_mesh_view* m)
{
  if (!m)
    invalid("null mesh");
  fbh::check_dim(m->dim);
  if (m->num_vertices < 0 || m->num_elements < 0)
    invalid("negative mesh size");
  if (m->num_elements > 0 && (!m->cells || !m->vertices || m->num_vertices == 0))
    invalid("mesh has cells but no vertex or cell data");
  if (m->num_vertices > INT32_MAX)
    invalid("vertex count exceeds the int32 index range");
}

fbk::LaunchSpec spec_of(const fb_variant& v, bool from_g)
{
  fbk::LaunchSpec s;
  s.op = v.op;
  s.dim = v.dim;
  s.prec = v.cfg.precision;
  s.mode = v.cfg.mode;
  s.path = v.path;
  s.from_g = from_g ? 1 : 0;
  s.staged = v.cfg.store == FB_STORE_DIRECT ? 0 : v.cfg.store == FB_STORE_STAGED ? 1 : v.cfg.store == FB_STORE_TMA ? 2 : 3;
  return s;
}

}  // namespace

// ====================================================================== ABI
extern "C" {

int fb_abi_version(void) { return FB_ABI_VERSION; }
int fb_device_count(void) { return device_count(); }
int64_t fb_launch_counter(void) { return fbk::launch_counter().load(); }

int64_t fb_kernel_setups(int device)
{
  if (device < 0 || device >= fbk::kMaxDevices)
    return -1;
  return fbk::device_setup_counters()[device].load();
}

int fb_release_workspace(int device, fb_error* err)
{
  return guarded(err,
                 [&]
                 {
                   DeviceGuard keep_device;
                   std::vector<std::pair<int, DeviceCtx*>> todo;
                   {
                     std::lock_guard<std::mutex> lock(g_ctx_mu);
                     for (auto& [d, c] : contexts())
                       if (device < 0 || d == device)
                         todo.emplace_back(d, c.get());
                   }
                   for (auto& [d, c] : todo)
                   {
                     std::lock_guard<std::mutex> lock(c->mu);
                     if (!c->ready)
                       continue;
                     cuda_check(cudaSetDevice(d), "cudaSetDevice");
                     cuda_check(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
                     c->release();
                   }
                 });
}

int fb_shard_bounds(int64_t num_slots, int parts, int64_t* bounds, fb_error* err)
{
  return guarded(err,
                 [&]
                 {
                   if (!bounds)
                     invalid("null bounds buffer");
                   const std::vector<int64_t> b = shard_bounds(num_slots, parts);
                   std::copy(b.begin(), b.end(), bounds);
                 });
}

int fb_krows(int op, int dim)
{
  if (op < 0 || op > 2 || (dim != 2 && dim != 3))
    return -1;
  return fbh::krows(op, dim);
}

int64_t fb_k_len(int op, int dim)
{
  if (op < 0 || op > 2 || (dim != 2 && dim != 3))
    return -1;
  return fbh::k_len(op, dim);
}

// src/engine.cpp:378-387
int64_t fb_flop_count(int op, int dim, int64_t ne)
{
  if (op < 0 || op > 2 || (dim != 2 && dim != 3))
    return -1;
  const int64_t kr = fbh::krows(op, dim), dd = static_cast<int64_t>(dim) * dim;
  if (op != FB_WEIGHTED_LAPLACIAN)
    return ne * kr * kr * 2 * dd;
  return ne * kr * kr * (dim + 1) * (2 * dd + 2);
}

// src/engine.cpp:287-299: batch / serial step / concurrent slot decomposition,
// which collapses to element*krows^2 + i + j*krows for every (bs, ce).
int64_t fb_element_matrix_index(int krows, int bs, int ce, int64_t element, int i, int j)
{
  if (krows < 1 || bs < 1 || ce < 1 || bs % ce != 0)
    return -1;
  const int64_t nk = static_cast<int64_t>(krows) * krows;
  const int64_t batch = element / bs;
  const int64_t within = element % bs;
  return batch * bs * nk + (within / ce) * ce * nk + (within % ce) * nk + i + static_cast<int64_t>(j) * krows;
}

int64_t fb_store_length(int op, int dim, int64_t ne, int bs)
{
  if (op < 0 || op > 2 || (dim != 2 && dim != 3) || bs < 1 || ne < 0)
    return -1;
  return store_len(fbh::krows(op, dim), ne, bs);
}

int fb_build_analytic_tensor(int op, int dim, double* k_out, int64_t k_len, fb_error* err)
{
  return guarded(err,
                 [&]
                 {
                   const std::vector<double> k = fbh::build_analytic_tensor(op, dim);
                   if (k_len != static_cast<int64_t>(k.size()))
                     invalid("analytic tensor buffer has the wrong length");
                   std::copy(k.begin(), k.end(), k_out);
                 });
}

int fb_structured_mesh_sizes(int dim, int n, int64_t* nv, int64_t* ne)
{
  try
  {
    fbh::structured_mesh_sizes(dim, n, *nv, *ne);
    return FB_OK;
  }
  catch (...)
  {
    return FB_ERR_INVALID_ARGUMENT;
  }
}

int fb_structured_mesh(int dim, int n, double* vertices, int32_t* cells, fb_error* err)
{
  return guarded(err, [&] { fbh::structured_mesh(dim, n, vertices, cells); });
}

int fb_jitter_mesh(int dim, double* vertices, int64_t nv, const int32_t* cells, int64_t ne,
                   double magnitude, uint64_t seed, fb_error* err)
{
  return guarded(err,
                 [&]
                 {
                   try
                   {
                     fbh::jitter_mesh(dim, vertices, nv, cells, ne, magnitude, seed);
                   }
                   catch (const std::runtime_error& e)
                   {
                     const std::string m = e.what();
                     const auto at = m.rfind(' ');
                     throw_code(FB_ERR_RUNTIME, m, std::stoll(m.substr(at + 1)));
                   }
                 });
}

// src/engine.cpp:301-337
fb_variant* fb_specialize(int op, int dim, const double* k_blocks, int64_t k_len,
                          const fb_kernel_config* config, fb_error* err)
{
  fb_variant* out = nullptr;
  guarded(err,
          [&]
          {
            if (op < 0 || op > 2)
              invalid("unknown operator");
            fbh::check_dim(dim);
            if (!config)
              invalid("null kernel config");
            validate_config(*config);
            if (!k_blocks || k_len != fbh::k_len(op, dim))
              invalid("analytic tensor was built for a different form");
            const int kr = fbh::krows(op, dim);
            const int64_t group = static_cast<int64_t>(kr) * kr * config->num_concurrent_elements;
            if (group > 1024)
              invalid("work-group bound exceeded: krows^2 * num_concurrent_elements = "
                      + std::to_string(group) + " > 1024");
            auto v = std::make_unique<fb_variant>();
            v->op = op;
            v->dim = dim;
            v->nb = dim + 1;
            v->krows = kr;
            v->ncoef = fbh::ncoef(op, dim);
            v->cfg = *config;
            v->k.assign(k_blocks, k_blocks + k_len);
            if (config->precision == FB_F32)
              analyse_k<float>(*v);
            else
              analyse_k<double>(*v);
            v->description = "bs" + std::to_string(config->element_batch_size) + "_ce"
                             + std::to_string(config->num_concurrent_elements);
            if (config->interleave_stores)
              v->description += "_is";
            if (config->loop_unroll)
              v->description += "_unroll";
            out = v.release();
          });
  return out;
}

void fb_variant_free(fb_variant* v) { delete v; }
const char* fb_variant_description(const fb_variant* v) { return v ? v->description.c_str() : ""; }
int fb_variant_path(const fb_variant* v) { return v ? v->path : -1; }

int fb_integrate_mesh(const fb_variant* vp, const fb_mesh_view* mesh, const double* coefficients,
                      void* out, int64_t out_len, const int* devices, int ndev, fb_error* err)
{
  return guarded(err,
                 [&]
                 {
                   const fb_variant& v = checked(vp);
                   validate_mesh_view(mesh);
                   if (mesh->dim != v.dim)
                     invalid("geometry dimension does not match form");
                   validate_coefficients(v, mesh->num_elements, coefficients);
                   validate_out(v, (mesh->num_elements + v.cfg.element_batch_size - 1) / v.cfg.element_batch_size * v.cfg.element_batch_size, out, out_len);
                   if (ndev < 0)
                     invalid("worker count must be >= 1");
                   Job j;
                   j.kind = Kind::Mesh;
                   j.var = &v;
                   j.dim = v.dim;
                   j.prec = v.cfg.precision;
                   j.nb = v.nb;
                   j.nk = v.krows * v.krows;
                   j.nv = mesh->num_vertices;
                   j.ne = mesh->num_elements;
                   j.nslots = out_len / j.nk;
                   j.vtx = mesh->vertices;
                   j.cells = mesh->cells;
                   j.coeffs = coefficients;
                   j.out = out;
                   j.vtx_dev = pointer_device(j.vtx);
                   j.cells_dev = pointer_device(j.cells);
                   j.coeff_dev = pointer_device(j.coeffs);
                   j.out_dev = pointer_device(out);
                   j.spec = spec_of(v, false);
                   run_job(j, devices, ndev);
                 });
}

int fb_integrate_packed(const fb_variant* vp, int dim, const void* g, int64_t num_batches,
                        int64_t ne, const double* coefficients, void* out, int64_t out_len,
                        const int* devices, int ndev, fb_error* err)
{
  return guarded(err,
                 [&]
                 {
                   const fb_variant& v = checked(vp);
                   if (dim != v.dim)
                     invalid("geometry dimension does not match form");
                   const int bs = v.cfg.element_batch_size;
                   if (num_batches < 0 || ne < 0 || ne > num_batches * bs)
                     invalid("packed geometry holds fewer slots than elements");
                   validate_coefficients(v, ne, coefficients);
                   validate_out(v, num_batches * bs, out, out_len);
                   if (num_batches > 0 && !g)
                     invalid("null packed geometry");
                   Job j;
                   j.kind = Kind::Packed;
                   j.var = &v;
                   j.dim = v.dim;
                   j.prec = v.cfg.precision;
                   j.nb = v.nb;
                   j.nk = v.krows * v.krows;
                   j.ne = ne;
                   j.nslots = num_batches * bs;
                   j.g = g;
                   j.coeffs = coefficients;
                   j.out = out;
                   j.g_dev = pointer_device(g);
                   j.coeff_dev = pointer_device(coefficients);
                   j.out_dev = pointer_device(out);
                   j.spec = spec_of(v, true);
                   run_job(j, devices, ndev);
                 });
}

int fb_pack_geometry(const fb_mesh_view* mesh, int bs, int precision, void* g_out, int64_t g_len,
                     const int* devices, int ndev, fb_error* err)
{
  return guarded(err,
                 [&]
                 {
                   validate_mesh_view(mesh);
                   if (bs < 1)
                     invalid("element_batch_size must be positive");
                   if (precision != FB_F32 && precision != FB_F64)
                     invalid("unknown precision");
                   const int dd = mesh->dim * mesh->dim;
                   const int64_t nslots = (mesh->num_elements + bs - 1) / bs * bs;
                   if (g_len != nslots * dd)
                     invalid("geometry buffer holds " + std::to_string(g_len) + " scalars; packing needs "
                             + std::to_string(nslots * dd));
                   Job j;
                   j.kind = Kind::Pack;
                   j.dim = mesh->dim;
                   j.prec = precision;
                   j.nb = mesh->dim + 1;
                   j.nk = dd;
                   j.nv = mesh->num_vertices;
                   j.ne = mesh->num_elements;
                   j.nslots = nslots;
                   j.vtx = mesh->vertices;
                   j.cells = mesh->cells;
                   j.out = g_out;
                   j.vtx_dev = pointer_device(j.vtx);
                   j.cells_dev = pointer_device(j.cells);
                   j.out_dev = pointer_device(g_out);
                   run_job(j, devices, ndev);
                 });
}

void* fb_device_alloc(int64_t bytes, int device, fb_error* err)
{
  void* p = nullptr;
  guarded(err,
          [&]
          {
            if (bytes < 0)
              invalid("negative allocation size");
            if (device_count() == 0)
              throw_code(FB_ERR_NO_DEVICE, "no CUDA device available");
            if (device < 0 || device >= device_count())
              invalid("device " + std::to_string(device) + " does not exist");
            int cur = 0;
            cuda_check(cudaGetDevice(&cur), "cudaGetDevice");
            cuda_check(cudaSetDevice(device), "cudaSetDevice");
            const cudaError_t e = cudaMalloc(&p, std::max<int64_t>(bytes, 1));
            cudaSetDevice(cur);
            cuda_check(e, "cudaMalloc");
          });
  return p;
}

int fb_free(void* device_ptr, fb_error* err)
{
  return guarded(err,
                 [&]
                 {
                   if (device_ptr)
                     cuda_check(cudaFree(device_ptr), "cudaFree");
                 });
}

int fb_pack_geometry_async(const fb_mesh_view* mesh, int bs, int precision, void* g_out, int64_t g_len,
                           int64_t* status, void* stream, fb_error* err)
{
  return guarded(err,
                 [&]
                 {
                   validate_mesh_view(mesh);
                   if (bs < 1)
                     invalid("element_batch_size must be positive");
                   if (precision != FB_F32 && precision != FB_F64)
                     invalid("unknown precision");
                   const int dd = mesh->dim * mesh->dim;
                   const int64_t nslots = (mesh->num_elements + bs - 1) / bs * bs;
                   if (g_len != nslots * dd)
                     invalid("geometry buffer holds " + std::to_string(g_len) + " scalars; packing needs "
                             + std::to_string(nslots * dd));
                   if (!status)
                     invalid("null status buffer");
                   if (nslots == 0)
                     return;
                   fbk::LaunchArgs a{};
                   a.vtx = mesh->vertices;
                   a.cells = mesh->cells;
                   a.out = g_out;
                   a.status = reinterpret_cast<long long*>(status);
                   a.nv = mesh->num_vertices;
                   a.ne = mesh->num_elements;
                   a.cells_aligned16 = aligned16(a.cells);
                   a.vtx_aligned16 = aligned16(a.vtx);
                   a.slot0 = 0;
                   a.nloc = nslots;
                   launch_pack_chunked(mesh->dim, precision, a, static_cast<cudaStream_t>(stream));
                 });
}

int fb_integrate_mesh_async(const fb_variant* vp, const fb_mesh_view* mesh, const double* coefficients,
                            void* out, int64_t out_len, int64_t* status, void* stream, fb_error* err)
{
  return guarded(err,
                 [&]
                 {
                   const fb_variant& v = checked(vp);
                   validate_mesh_view(mesh);
                   if (mesh->dim != v.dim)
                     invalid("geometry dimension does not match form");
                   validate_coefficients(v, mesh->num_elements, coefficients);
                   validate_out(v, (mesh->num_elements + v.cfg.element_batch_size - 1) / v.cfg.element_batch_size * v.cfg.element_batch_size, out, out_len);
                   if (!status)
                     invalid("null status buffer");
                   int dev = 0;
                   cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
                   fbk::LaunchArgs a{};
                   a.vtx = mesh->vertices;
                   a.cells = mesh->cells;
                   a.coeffs = coefficients;
                   a.out = out;
                   a.kdense = kdense_on(v, dev);
                   a.status = reinterpret_cast<long long*>(status);
                   a.nv = mesh->num_vertices;
                   a.ne = mesh->num_elements;
                   a.nloc = out_len / (v.krows * v.krows);
                   a.slot0 = 0;
                   a.cells_aligned16 = aligned16(a.cells);
                   a.vtx_aligned16 = aligned16(a.vtx);
                   fbk::LaunchSpec s = spec_of(v, false);
                   if (!aligned16(out))
                     s.staged = 0;
                   launch_integrate_chunked(s, a, v.kp, v.krows * v.krows, v.dim * v.dim,
                                            scalar_size(v.cfg.precision), static_cast<cudaStream_t>(stream));
                 });
}

int fb_integrate_packed_async(const fb_variant* vp, int dim, const void* g, int64_t num_batches,
                              int64_t ne, const double* coefficients, void* out, int64_t out_len,
                              void* stream, fb_error* err)
{
  return guarded(err,
                 [&]
                 {
                   const fb_variant& v = checked(vp);
                   if (dim != v.dim)
                     invalid("geometry dimension does not match form");
                   if (num_batches < 0 || ne < 0 || ne > num_batches * v.cfg.element_batch_size)
                     invalid("packed geometry holds fewer slots than elements");
                   validate_coefficients(v, ne, coefficients);
                   validate_out(v, num_batches * v.cfg.element_batch_size, out, out_len);
                   int dev = 0;
                   cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
                   fbk::LaunchArgs a{};
                   a.g_in = g;
                   a.coeffs = coefficients;
                   a.out = out;
                   a.kdense = kdense_on(v, dev);
                   a.ne = ne;
                   a.nloc = num_batches * v.cfg.element_batch_size;
                   fbk::LaunchSpec s = spec_of(v, true);
                   if (!aligned16(out))
                     s.staged = 0;
                   launch_integrate_chunked(s, a, v.kp, v.krows * v.krows, v.dim * v.dim,
                                            scalar_size(v.cfg.precision), static_cast<cudaStream_t>(stream));
                 });
}

int fb_status_reset(int64_t* status, void* stream, fb_error* err)
{
  return guarded(err,
                 [&]
                 {
                   cuda_check(cudaMemsetAsync(status, 0x7f, 2 * sizeof(int64_t),
                                              static_cast<cudaStream_t>(stream)),
                              "cudaMemsetAsync");
                 });
}

int fb_status_check(const int64_t* status, void* stream, fb_error* err)
{
  return guarded(err,
                 [&]
                 {
                   long long w[2];
                   cuda_check(cudaMemcpyAsync(w, status, sizeof w, cudaMemcpyDeviceToHost,
                                              static_cast<cudaStream_t>(stream)),
                              "download status");
                   cuda_check(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)),
                              "cudaStreamSynchronize");
                   check_status_words(w);
                 });
}

}  // extern "C"
