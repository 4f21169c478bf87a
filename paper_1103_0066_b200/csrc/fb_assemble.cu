// fb_assemble.cu -- global CSR assembly from the element-matrix store
// (the reference stops at element matrices).
//
// Deterministic gather, no atomics.  A warp owns 32 consecutive vertices and
// one component pair (ci, cj); lane l walks vertex v = 32g + l's incident
// elements in ascending element order (sliced SELL-32 lists: every lane
// load of the plan is coalesced) and adds row a (v's local index),
// component block (ci, cj), of each element matrix into per-neighbour
// accumulators in shared memory ([slot][thread], conflict-free).  Every CSR
// entry thus receives its contributions in ascending element order from +0
// -- bitwise the serial element loop of the oracle (oracle/fb_oracle.c
// fbo_assemble).  When the variant's element matrices are bitwise symmetric
// (the sparse-symmetric kernel paths mirror one triangle) the row is read as
// the contiguous column (one 16-byte load in 3D f32).  Incidences are
// processed U at a time so a lane has U element rows in flight.  Vertices
// with more than kAsmSlots neighbours accumulate directly in their own
// (thread-private) rows of the output.
#include <atomic>
#include <cstdint>

#include <cuda_runtime.h>

#include "fb_internal.h"

namespace fbk {

std::atomic<long long>& launch_counter();

namespace {

constexpr int kAsmWarps = 4;
constexpr int kAsmThreads = 32 * kAsmWarps;
constexpr int kAsmSlots = 32;  // neighbours held in shared memory per thread
#ifndef FB_ASM_U
#define FB_ASM_U 8
#endif
constexpr int kAsmUnroll = FB_ASM_U;  // incidences in flight per lane
constexpr uint32_t kPad = 0xffffffffu;

template <class S>
__device__ __forceinline__ S add_rn(S a, S b);
template <>
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
template <>
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }

// The NB entries of element-matrix row i = aa + ci*NB, columns b + cj*NB.
template <class S, int NB, int KROWS, bool SYM>
__device__ __forceinline__ void load_row(const S* blk, int i, int cj, S (&r)[NB])
{
  if constexpr (SYM)
  {
    // A(i, j) == A(j, i): the contiguous column i, rows cj*NB .. cj*NB+NB-1
    const S* p = blk + cj * NB + i * KROWS;
    if constexpr (NB == 4 && sizeof(S) == 4)
    {
      const float4 q = __ldg(reinterpret_cast<const float4*>(p));
      r[0] = q.x;
      r[1] = q.y;
      r[2] = q.z;
      r[NB - 1] = q.w;
    }
    else if constexpr (NB == 4 && sizeof(S) == 8)
    {
      const double2 q0 = __ldg(reinterpret_cast<const double2*>(p));
      const double2 q1 = __ldg(reinterpret_cast<const double2*>(p) + 1);
      r[0] = q0.x;
      r[1] = q0.y;
      r[2] = q1.x;
      r[NB - 1] = q1.y;
    }
    else
    {
#pragma unroll
      for (int b = 0; b < NB; ++b)
        r[b] = __ldg(p + b);
    }
  }
  else
  {
#pragma unroll
    for (int b = 0; b < NB; ++b)
      r[b] = __ldg(blk + i + (b + cj * NB) * KROWS);
  }
}

template <class S, int DIM, int NC, bool SYM>
__global__ void __launch_bounds__(kAsmThreads) fb_assemble_kernel(const AsmArgs a)
{
  constexpr int NB = DIM + 1, KROWS = NB * NC, NK = KROWS * KROWS, NC2 = NC * NC;
  constexpr int U = kAsmUnroll;
  __shared__ S acc_s[kAsmSlots * kAsmThreads];
  S* acc = acc_s + threadIdx.x;
  S* vals = static_cast<S*>(a.values);
  const S* store = static_cast<const S*>(a.store);
  const int lane = threadIdx.x & 31;
  const int64_t ngroups = (a.nv + 31) / 32;
  const int64_t nwarps = ngroups * NC2;
  for (int64_t w = static_cast<int64_t>(blockIdx.x) * kAsmWarps + (threadIdx.x >> 5); w < nwarps;
       w += static_cast<int64_t>(gridDim.x) * kAsmWarps)
  {
    const int64_t g = w / NC2;
    const int cp = static_cast<int>(w - g * NC2);
    const int ci = cp / NC, cj = cp % NC;
    const int64_t v = g * 32 + lane;
    const bool live = v < a.nv;
    const int64_t r0 = live ? __ldg(a.nbr_ptr + v) : 0;
    const int deg = live ? static_cast<int>(__ldg(a.nbr_ptr + v + 1) - r0) : 0;
    const int64_t row = r0 * NC2 + static_cast<int64_t>(ci) * deg * NC + cj;  // + k*NC
    const bool in_smem = deg <= kAsmSlots;
    if (in_smem)
      for (int k = 0; k < deg; ++k)
        acc[k * kAsmThreads] = S(0);
    else
      for (int k = 0; k < deg; ++k)
        vals[row + static_cast<int64_t>(k) * NC] = S(0);
    const int64_t q0 = __ldg(a.goff + g), q1 = __ldg(a.goff + g + 1);
    for (int64_t q = q0 + lane; q < q1; q += 32 * U)
    {
      uint32_t pk[U], ps[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
      {
        const int64_t qu = q + 32 * u;
        pk[u] = qu < q1 ? __ldg(a.spk + qu) : kPad;
        ps[u] = qu < q1 ? __ldg(a.spos + qu) : 0u;
      }
      S r[U][NB];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (pk[u] != kPad)
        {
          const int64_t e = pk[u] >> 2;
          const int aa = static_cast<int>(pk[u] & 3u);
          load_row<S, NB, KROWS, SYM>(store + e * NK, aa + ci * NB, cj, r[u]);
        }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (pk[u] != kPad)
        {
#pragma unroll
          for (int b = 0; b < NB; ++b)
          {
            const int k = (ps[u] >> (8 * b)) & 0xffu;
            if (in_smem)
              acc[k * kAsmThreads] = add_rn(acc[k * kAsmThreads], r[u][b]);
            else
            {
              S* p = vals + row + static_cast<int64_t>(k) * NC;
              *p = add_rn(*p, r[u][b]);
            }
          }
        }
    }
    if (in_smem)
      for (int k = 0; k < deg; ++k)
        vals[row + static_cast<int64_t>(k) * NC] = acc[k * kAsmThreads];
  }
}

template <class S, int DIM, int NC, bool SYM>
cudaError_t go(const AsmArgs& a, cudaStream_t st)
{
  const int64_t nwarps = (a.nv + 31) / 32 * NC * NC;
  if (nwarps <= 0)
    return cudaSuccess;
  static int grid_cap = 0;
  if (grid_cap == 0)
  {
    int blocks = 0, dev = 0, sms = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, fb_assemble_kernel<S, DIM, NC, SYM>, kAsmThreads, 0);
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    grid_cap = (blocks > 0 ? blocks : 1) * (sms > 0 ? sms : 1);
  }
  const int64_t need = (nwarps + kAsmWarps - 1) / kAsmWarps;
  const unsigned grid = static_cast<unsigned>(need < grid_cap ? need : grid_cap);
  fb_assemble_kernel<S, DIM, NC, SYM><<<grid, kAsmThreads, 0, st>>>(a);
  launch_counter().fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

template <class S, int DIM, int NC>
cudaError_t go_sym(const AsmArgs& a, cudaStream_t st)
{
  return a.sym ? go<S, DIM, NC, true>(a, st) : go<S, DIM, NC, false>(a, st);
}

}  // namespace

cudaError_t launch_assemble(int dim, int nc, int prec, const AsmArgs& a, cudaStream_t st)
{
  if (prec == 0)
  {
    if (dim == 2)
      return nc == 1 ? go_sym<float, 2, 1>(a, st) : go_sym<float, 2, 2>(a, st);
    return nc == 1 ? go_sym<float, 3, 1>(a, st) : go_sym<float, 3, 3>(a, st);
  }
  if (dim == 2)
    return nc == 1 ? go_sym<double, 2, 1>(a, st) : go_sym<double, 2, 2>(a, st);
  return nc == 1 ? go_sym<double, 3, 1>(a, st) : go_sym<double, 3, 3>(a, st);
}

}  // namespace fbk
