// fb_assemble_g.cu -- global CSR assembly straight from the packed geometry
// (G, reference PackedGeometry layout): the element matrices are never
// stored.  Same plan, same deterministic per-vertex gather as fb_assemble.cu,
// but each incidence's element-matrix row is recomputed in registers from
// G_e with the G-input integration path's own contraction (contract_sparse,
// fb_kernels.cuh; same arithmetic mode, no symmetric shortcut), so every
// contribution has the bits integrate_batches would have stored and the sum
// order is the same ascending element order: the values are bitwise those of
// assembling the integrate_batches store.  For elasticity only the c_i == c_j
// component blocks are added (the others are +0, an identity for an
// accumulator that starts at +0 and is never -0).
//
// Bytes per element: G (dim^2 scalars) read once per incidence instead of an
// element-matrix row, and no store written -- the win grows with krows^2
// (3D elasticity: 36 B of G vs a 576 B matrix).  In 3D an incidence with
// local index a != 0 reads only row a-1 of G and contracts the one row it
// needs (contract_row); the CSR row block leaves with 32-byte full-sector
// stores (fb_asm_store.cuh).
#include <atomic>
#include <cstdint>

#include <cuda_runtime.h>

#include "fb_asm_store.cuh"
#include "fb_devcache.h"
#include "fb_kernels.cuh"

namespace fbk {

std::atomic<long long>& launch_counter();

namespace {

constexpr uint32_t kPadG = 0xffffffffu;

#ifndef FB_ASMG_U
#define FB_ASMG_U 4
#endif
#ifndef FB_ASMG_EVL
#define FB_ASMG_EVL 0  // G loads under an L2 evict_last policy (A/B: neutral to -7 %, off)
#endif
template <class T>
__device__ __forceinline__ T ldg_g(const T* p)
{
  if constexpr (FB_ASMG_EVL)
    return ld_el(p);
  else
    return __ldg(p);
}
#ifndef FB_ASMG_VEC
#define FB_ASMG_VEC 1
#endif

template <class S>
__device__ __forceinline__ S add_rn_g(S a, S b);
template <>
__device__ __forceinline__ float add_rn_g(float a, float b) { return __fadd_rn(a, b); }
template <>
__device__ __forceinline__ double add_rn_g(double a, double b) { return __dadd_rn(a, b); }

template <class S, int DIM, int OP>
struct GShape {
  static constexpr int NC = OP == kElasticity ? DIM : 1;
  static constexpr int WARPS = 4;
  // neighbours accumulated in shared memory (<= 48 KB static)
  static constexpr int FIT = 48 * 1024 / (32 * WARPS * static_cast<int>(sizeof(S)));
  static constexpr int SLOTS = FIT < 32 ? FIT : 32;
  static constexpr int U = FB_ASMG_U;  // incidences in flight per lane
};

// G_e (DD scalars at gin + e*DD, 4-byte aligned only for 3D f32) with the
// fewest 16-byte loads: the aligned 16-byte words covering it, then a
// register select by the misalignment.  The element whose covering words
// would run past the end of G (ng scalars) is read scalar-wise, and all of
// G when it is not 16-byte aligned (ng < 0).
template <class S, int DD>
__device__ __forceinline__ void load_g(const S* gin, int64_t e, int64_t ng, S (&g)[DD])
{
  constexpr int W = 16 / static_cast<int>(sizeof(S));  // scalars per 16-byte word
  const int64_t first = e * DD;
  if (!FB_ASMG_VEC || ng < 0)  // ng < 0: G not 16-byte aligned
  {
#pragma unroll
    for (int t = 0; t < DD; ++t)
      g[t] = ldg_g(gin + first + t);
    return;
  }
  if constexpr (DD % W == 0)
  {
    // every G_e starts on a 16-byte boundary (G does)
#pragma unroll
    for (int t = 0; t < DD; t += W)
    {
      if constexpr (W == 4)
      {
        const float4 q = ldg_g(reinterpret_cast<const float4*>(gin + first + t));
        g[t] = q.x, g[t + 1] = q.y, g[t + 2] = q.z, g[t + 3] = q.w;
      }
      else
      {
        const double2 q = ldg_g(reinterpret_cast<const double2*>(gin + first + t));
        g[t] = q.x, g[t + 1] = q.y;
      }
    }
  }
  else
  {
    constexpr int NW = (DD + W - 1 + W - 1) / W;  // words covering any misalignment
    const int sh = static_cast<int>(first % W);
    const int64_t w0 = first - sh;
    if (w0 + NW * W > ng)
    {
#pragma unroll
      for (int t = 0; t < DD; ++t)
        g[t] = ldg_g(gin + first + t);
      return;
    }
    S c[NW * W];
#pragma unroll
    for (int k = 0; k < NW; ++k)
    {
      if constexpr (W == 4)
      {
        const float4 q = ldg_g(reinterpret_cast<const float4*>(gin + w0) + k);
        c[4 * k] = q.x, c[4 * k + 1] = q.y, c[4 * k + 2] = q.z, c[4 * k + 3] = q.w;
      }
      else
      {
        const double2 q = ldg_g(reinterpret_cast<const double2*>(gin + w0) + k);
        c[2 * k] = q.x, c[2 * k + 1] = q.y;
      }
    }
#pragma unroll
    for (int t = 0; t < DD; ++t)
    {
      S x = c[t];
#pragma unroll
      for (int r = 1; r < W; ++r)
        if (t + r < NW * W)
          x = sh == r ? c[t + r] : x;
      g[t] = x;
    }
  }
}

// Row aa (runtime) of the nb x nb Laplacian-like block, selected without
// dynamic register indexing.
template <class S, int NB>
__device__ __forceinline__ void select_row(const S (&vv)[NB * NB], int aa, S (&x)[NB])
{
#pragma unroll
  for (int b = 0; b < NB; ++b)
    x[b] = vv[b];
#pragma unroll
  for (int r = 1; r < NB; ++r)
#pragma unroll
    for (int b = 0; b < NB; ++b)
      x[b] = aa == r ? vv[r * NB + b] : x[b];
}

#ifndef FB_ASMG_ROW
#define FB_ASMG_ROW 1
#endif
// Row a != 0 (runtime) of contract_sparse<SYM = false>: on the P1 pattern
// only mu = a-1 contributes, so the row needs G's row a-1 (dim scalars)
// alone.  Same terms, same (c, mu, nu) order, same operations as
// contract_sparse, hence the same bits.
template <class S, int DIM, int OP, int MODE, bool UNI>
__device__ __forceinline__ void contract_row(const S (&gr)[DIM], const S (&w)[DIM + 1], const KP<S, DIM, OP>& kp,
                                             int a, S (&x)[DIM + 1])
{
  using Sh = Shape<DIM, OP>;
  using A = Ar<S, MODE>;
  constexpr int NB = DIM + 1, NC = Sh::NC, DD = Sh::DD;
  S m[UNI ? NC * DIM : 1];
  if (UNI)
  {
#pragma unroll
    for (int c = 0; c < NC; ++c)
#pragma unroll
      for (int nu = 0; nu < DIM; ++nu)
        m[UNI ? c * DIM + nu : 0] = OP == kWeighted ? A::mul(A::mul(w[c], gr[nu]), kp.k[c]) : A::mul(gr[nu], kp.k[c]);
  }
#pragma unroll
  for (int b = 0; b < NB; ++b)
  {
    S acc = S(0);
#pragma unroll
    for (int c = 0; c < NC; ++c)
#pragma unroll
      for (int nu = 0; nu < DIM; ++nu)
      {
        if (b != 0 && nu != b - 1)
          continue;
        if (UNI)
        {
          const S p = m[UNI ? c * DIM + nu : 0];
          acc = A::add(acc, b == 0 ? -p : p);  // sigma_ab = -1 iff b == 0 (a != 0)
        }
        else
        {
          const S kv = kp.k[((a * NB + b) * NC + c) * DD + (a - 1) * DIM + nu];
          if (OP == kWeighted)
            acc = A::mac(acc, A::mul(w[c], gr[nu]), kv);
          else
            acc = A::mac(acc, gr[nu], kv);
        }
      }
    x[b] = acc;
  }
}

// A warp owns 32 consecutive vertices and all their rows.  Elasticity: the
// element matrix is block diagonal with nc copies of the Laplacian-like
// block, so the nc diagonal component blocks of a CSR row block receive the
// same additions in the same order: one accumulator per neighbour, written
// to the nc diagonal entries; the off-diagonal entries are written as +0.
template <class S, int DIM, int OP, int MODE, bool UNI>
__global__ void __launch_bounds__(32 * GShape<S, DIM, OP>::WARPS)
    fb_assemble_g_kernel(const AsmArgs a, const __grid_constant__ KP<S, DIM, OP> kp)
{
  using G = GShape<S, DIM, OP>;
  constexpr int NB = DIM + 1, NC = G::NC, DD = DIM * DIM;
  constexpr int T = 32 * G::WARPS, SLOTS = G::SLOTS, U = G::U;
  // row-only contraction for a != 0: 3D (A/B: 3D-E f32 0.43 -> 0.38 ms, f64
  // 0.74 -> 0.61, 3D-L f32 0.65 -> 0.53); 2D loses ~5 % (2D-E 0.033 -> 0.035)
  constexpr bool ROWP = FB_ASMG_ROW && DIM == 3;
  __shared__ S acc_s[SLOTS * T];
  S* acc = acc_s + threadIdx.x;
  S* vals = static_cast<S*>(a.values);
  const S* gin = static_cast<const S*>(a.g_in);
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (a.nv + 31) / 32;
  for (int64_t g = static_cast<int64_t>(blockIdx.x) * (T / 32) + (threadIdx.x >> 5); g < nwarps;
       g += static_cast<int64_t>(gridDim.x) * (T / 32))
  {
    const int64_t v = g * 32 + lane;
    const bool live = v < a.nv;
    const int64_t r0 = live ? __ldg(a.nbr_ptr + v) : 0;
    const int deg = live ? static_cast<int>(__ldg(a.nbr_ptr + v + 1) - r0) : 0;
    // CSR row (v, ci) starts at r0*NC*NC + ci*deg*NC; entry (k, cj) at + k*NC + cj.
    const int64_t row0 = r0 * NC * NC;
    const bool in_smem = deg <= SLOTS;
    const int64_t q0 = __ldg(a.goff + g), q1 = __ldg(a.goff + g + 1);
    uint32_t pk[U], ps[U];
    auto load_plan = [&](int64_t q, uint32_t (&k)[U], uint32_t (&p)[U])
    {
#pragma unroll
      for (int u = 0; u < U; ++u)
      {
        const int64_t qu = q + 32 * u;
        k[u] = qu < q1 ? __ldg(a.spk + qu) : kPadG;
        p[u] = qu < q1 ? __ldg(a.spos + qu) : 0u;
      }
    };
    load_plan(q0 + lane, pk, ps);
    if (in_smem)
      for (int k = 0; k < deg; ++k)
        acc[k * T] = S(0);
    else
      for (int k = 0; k < deg * NC * NC; ++k)
        vals[row0 + k] = S(0);
    for (int64_t q = q0 + lane; q < q1; q += 32 * U)
    {
      uint32_t npk[U], nps[U];
      load_plan(q + 32 * U, npk, nps);
      S ge[U][DD];
      S we[U][DIM + 1];
#pragma unroll
      for (int u = 0; u < U; ++u)
      {
        const int64_t e = pk[u] != kPadG ? (pk[u] >> 2) : 0;
        const int aa = static_cast<int>(pk[u] & 3u);
        if (pk[u] != kPadG)
        {
          if (!ROWP || aa == 0)
            load_g<S, DD>(gin, e, a.g_len, ge[u]);
          else  // row a-1 of G only
          {
#pragma unroll
            for (int nu = 0; nu < DIM; ++nu)
              ge[u][nu] = ldg_g(gin + e * DD + (aa - 1) * DIM + nu);
          }
        }
#pragma unroll
        for (int c = 0; c <= DIM; ++c)
          we[u][c] = OP == kWeighted && pk[u] != kPadG ? static_cast<S>(__ldg(a.coeffs + e * (DIM + 1) + c)) : S(0);
      }
      // one incidence at a time: two incidences may share a neighbour
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (pk[u] != kPadG)
        {
          const int aa = static_cast<int>(pk[u] & 3u);
          S x[NB];
          if (!ROWP)
          {
            S vv[NB * NB];
            contract_sparse<S, DIM, OP, MODE, false, UNI>(ge[u], we[u], kp, vv);
            select_row<S, NB>(vv, aa, x);
          }
          else if (aa == 0)
          {
            S vv[NB * NB];
            contract_sparse<S, DIM, OP, MODE, false, UNI>(ge[u], we[u], kp, vv);
#pragma unroll
            for (int b = 0; b < NB; ++b)
              x[b] = vv[b];
          }
          else
          {
            S gr[DIM];
#pragma unroll
            for (int nu = 0; nu < DIM; ++nu)
              gr[nu] = ge[u][nu];
            contract_row<S, DIM, OP, MODE, UNI>(gr, we[u], kp, aa, x);
          }
#pragma unroll
          for (int b = 0; b < NB; ++b)
          {
            const int k = static_cast<int>((ps[u] >> (8 * b)) & 0xffu);
            if (in_smem)
              acc[k * T] = add_rn_g(acc[k * T], x[b]);
            else
            {
              // global accumulation in the (v, 0) row block; copied to the
              // other diagonal blocks at the end
              S* p = vals + row0 + k * NC;
              *p = add_rn_g(*p, x[b]);
            }
          }
        }
#pragma unroll
      for (int u = 0; u < U; ++u)
      {
        pk[u] = npk[u];
        ps[u] = nps[u];
      }
    }
    if (in_smem)
      write_block<S, NC, T, FB_ASMG_VECST != 0>(vals + row0, deg, acc);
    else if (NC > 1)
      for (int k = 0; k < deg; ++k)
      {
        const S x = vals[row0 + k * NC];
#pragma unroll
        for (int ci = 1; ci < NC; ++ci)
          vals[row0 + static_cast<int64_t>(ci) * deg * NC + k * NC + ci] = x;
      }
  }
}

template <class S, int DIM, int OP, int MODE, bool UNI>
cudaError_t go_g(const AsmArgs& a, const KParamBlob& kb, cudaStream_t st)
{
  using G = GShape<S, DIM, OP>;
  constexpr int T = 32 * G::WARPS;
  const int64_t nwarps = (a.nv + 31) / 32;
  if (nwarps <= 0)
    return cudaSuccess;
  // resident CTAs per SM x SMs, computed once per instantiation and device
  // (fb_devcache.h; reentrant: concurrent first calls compute the same value)
  static PerDevice grid_cap_cache;
  int dev = 0;
  cudaGetDevice(&dev);
  const int grid_cap = grid_cap_cache.get(
      dev,
      [&]
      {
        int blocks = 0, sms = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, fb_assemble_g_kernel<S, DIM, OP, MODE, UNI>, T, 0);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        return (blocks > 0 ? blocks : 1) * (sms > 0 ? sms : 1);
      },
      device_setup_counters());
  const int64_t need = (nwarps + T / 32 - 1) / (T / 32);
  const unsigned grid = static_cast<unsigned>(need < grid_cap ? need : grid_cap);
  const KP<S, DIM, OP>& kp = *reinterpret_cast<const KP<S, DIM, OP>*>(kb.bytes);
  fb_assemble_g_kernel<S, DIM, OP, MODE, UNI><<<grid, T, 0, st>>>(a, kp);
  launch_counter().fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

template <class S, int DIM, int OP>
cudaError_t go_g_mode(const LaunchSpec& s, const AsmArgs& a, const KParamBlob& kb, cudaStream_t st)
{
  const bool uni = s.path == kUniformSym;
  if (s.mode == kFast)
    return uni ? go_g<S, DIM, OP, kFast, true>(a, kb, st) : go_g<S, DIM, OP, kFast, false>(a, kb, st);
  return uni ? go_g<S, DIM, OP, kStrict, true>(a, kb, st) : go_g<S, DIM, OP, kStrict, false>(a, kb, st);
}

template <class S, int DIM>
cudaError_t go_g_op(const LaunchSpec& s, const AsmArgs& a, const KParamBlob& kb, cudaStream_t st)
{
  switch (s.op)
  {
  case kLaplacian:
    return go_g_mode<S, DIM, kLaplacian>(s, a, kb, st);
  case kElasticity:
    return go_g_mode<S, DIM, kElasticity>(s, a, kb, st);
  default:
    return go_g_mode<S, DIM, kWeighted>(s, a, kb, st);
  }
}

}  // namespace

// s.path must be a sparse path (the dense fallback has no G-input assembly)
cudaError_t launch_assemble_g(const LaunchSpec& s, const AsmArgs& a, const KParamBlob& kb, cudaStream_t st)
{
  if (s.prec == 0)
    return s.dim == 2 ? go_g_op<float, 2>(s, a, kb, st) : go_g_op<float, 3>(s, a, kb, st);
  return s.dim == 2 ? go_g_op<double, 2>(s, a, kb, st) : go_g_op<double, 3>(s, a, kb, st);
}

}  // namespace fbk
