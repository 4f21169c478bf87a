// fb_assemble.cu -- global CSR assembly from the element-matrix store
// (the reference stops at element matrices).
//
// Deterministic gather, no atomics: one thread per (vertex v, component pair
// (ci, cj)).  It walks v's incident elements in ascending element order and
// adds row a (v's local index) of each element matrix, component block
// (ci, cj), into per-neighbour accumulators held in shared memory
// ([slot][thread], conflict-free).  Every CSR entry therefore receives its
// contributions in ascending element order from +0 -- bitwise the serial
// element loop of the oracle (oracle/fb_oracle.c fbo_assemble).  Vertices
// with more than kAsmSlots neighbours accumulate directly in their own
// (thread-private) rows of the output instead.
//
// HBM traffic per call: the incidence lists (4 + nb bytes per incidence, nb
// incidences per element), the store's real elements (read once from HBM;
// the nb readers of an element are nearby vertices and meet in L2), and the
// CSR values written once.
#include <atomic>
#include <cstdint>

#include <cuda_runtime.h>

#include "fb_internal.h"

namespace fbk {

std::atomic<long long>& launch_counter();

namespace {

constexpr int kAsmThreads = 128;
constexpr int kAsmSlots = 32;  // neighbours held in shared memory per thread

template <class S>
__device__ __forceinline__ S add_rn(S a, S b);
template <>
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
template <>
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }

template <class S, int DIM, int NC>
__global__ void __launch_bounds__(kAsmThreads) fb_assemble_kernel(const AsmArgs a)
{
  constexpr int NB = DIM + 1, KROWS = NB * NC, NK = KROWS * KROWS, NC2 = NC * NC;
  __shared__ S acc_s[kAsmSlots * kAsmThreads];
  const int64_t nthreads = a.nv * NC2;
  S* vals = static_cast<S*>(a.values);
  const S* store = static_cast<const S*>(a.store);
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * kAsmThreads + threadIdx.x; t < nthreads;
       t += static_cast<int64_t>(gridDim.x) * kAsmThreads)
  {
    const int64_t v = t / NC2;
    const int cp = static_cast<int>(t - v * NC2);
    const int ci = cp / NC, cj = cp % NC;
    const int64_t r0 = __ldg(a.nbr_ptr + v);
    const int deg = static_cast<int>(__ldg(a.nbr_ptr + v + 1) - r0);
    const int64_t row = r0 * NC2 + static_cast<int64_t>(ci) * deg * NC + cj;  // + k*NC
    const bool in_smem = deg <= kAsmSlots;
    S* acc = in_smem ? acc_s + threadIdx.x : vals + row;
    const int step = in_smem ? kAsmThreads : NC;
    for (int k = 0; k < deg; ++k)
      acc[k * step] = S(0);
    const int64_t q1 = __ldg(a.v2e_ptr + v + 1);
    for (int64_t q = __ldg(a.v2e_ptr + v); q < q1; ++q)
    {
      const uint32_t pk = __ldg(a.v2e + q);
      const int64_t e = pk >> 2;
      const int aa = static_cast<int>(pk & 3u);
      // row i = aa + ci*NB of element e; column j = b + cj*NB
      const S* blk = store + e * NK + aa + ci * NB + cj * NB * KROWS;
      int pos[NB];
      if (NB == 4)
      {
        const uint32_t w = __ldg(reinterpret_cast<const uint32_t*>(a.nbrpos) + q);
#pragma unroll
        for (int b = 0; b < NB; ++b)
          pos[b] = (w >> (8 * b)) & 0xffu;
      }
      else
      {
#pragma unroll
        for (int b = 0; b < NB; ++b)
          pos[b] = __ldg(a.nbrpos + q * NB + b);
      }
#pragma unroll
      for (int b = 0; b < NB; ++b)
      {
        const S val = __ldg(blk + b * KROWS);
        S* p = acc + pos[b] * step;
        *p = add_rn(*p, val);
      }
    }
    if (in_smem)
      for (int k = 0; k < deg; ++k)
        vals[row + static_cast<int64_t>(k) * NC] = acc[k * kAsmThreads];
  }
}

template <class S, int DIM, int NC>
cudaError_t go(const AsmArgs& a, cudaStream_t st)
{
  const int64_t n = a.nv * NC * NC;
  if (n <= 0)
    return cudaSuccess;
  static int grid_cap = 0;
  if (grid_cap == 0)
  {
    int blocks = 0, dev = 0, sms = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, fb_assemble_kernel<S, DIM, NC>, kAsmThreads, 0);
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    grid_cap = (blocks > 0 ? blocks : 1) * (sms > 0 ? sms : 1) * 8;
  }
  const int64_t need = (n + kAsmThreads - 1) / kAsmThreads;
  const unsigned grid = static_cast<unsigned>(need < grid_cap ? need : grid_cap);
  fb_assemble_kernel<S, DIM, NC><<<grid, kAsmThreads, 0, st>>>(a);
  launch_counter().fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_assemble(int dim, int nc, int prec, const AsmArgs& a, cudaStream_t st)
{
  if (prec == 0)
  {
    if (dim == 2)
      return nc == 1 ? go<float, 2, 1>(a, st) : go<float, 2, 2>(a, st);
    return nc == 1 ? go<float, 3, 1>(a, st) : go<float, 3, 3>(a, st);
  }
  if (dim == 2)
    return nc == 1 ? go<double, 2, 1>(a, st) : go<double, 2, 2>(a, st);
  return nc == 1 ? go<double, 3, 1>(a, st) : go<double, 3, 3>(a, st);
}

}  // namespace fbk
