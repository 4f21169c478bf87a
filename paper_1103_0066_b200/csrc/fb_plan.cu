// fb_plan.cu -- the assembly plan built on the GPU (when the connectivity is
// device-resident): the same plan the host builder (fb_assembly.cpp) makes,
// array for array, so the assembled values do not depend on where the plan
// was built.
//
//   1. validate cells (lowest bad cell per error) and count incidences;
//   2. exclusive scan -> per-vertex incidence offsets;
//   3. scatter incidences with atomics, then sort each vertex's list
//      ascending in (e << 2 | a) -- deterministic whatever the atomic order;
//   4. per vertex, the sorted unique neighbour list (thread-local, <= 255)
//      -> degree; scan -> row-block offsets;
//   5. SELL-32 group widths (warp max) -> scan -> group offsets;
//   6. per vertex again: write the neighbour list and, per incidence, the
//      packed entry and the neighbour slots of the element's vertices.
#include <atomic>
#include <cstdint>

#include <cub/device/device_scan.cuh>
#include <cuda_runtime.h>

#include "fb_internal.h"

namespace fbk {

std::atomic<long long>& launch_counter();

namespace {

constexpr int kT = 256;
constexpr int kMaxDeg = 255;

unsigned blocks_for(int64_t n) { return static_cast<unsigned>((n + kT - 1) / kT); }

template <int NB>
__global__ void validate_count(const int32_t* __restrict__ cells, int64_t ne, int64_t nv,
                               unsigned long long* __restrict__ cnt, unsigned long long* __restrict__ bad)
{
  const int64_t e = blockIdx.x * static_cast<int64_t>(kT) + threadIdx.x;
  if (e >= ne)
    return;
  int v[NB];
  bool range_ok = true, distinct = true;
#pragma unroll
  for (int a = 0; a < NB; ++a)
  {
    v[a] = __ldg(cells + e * NB + a);
    range_ok &= v[a] >= 0 && v[a] < nv;
#pragma unroll
    for (int b = 0; b < a; ++b)
      distinct &= v[a] != v[b];
  }
  if (!range_ok)
    atomicMin(bad + 0, static_cast<unsigned long long>(e));
  else if (!distinct)
    atomicMin(bad + 1, static_cast<unsigned long long>(e));
  else
  {
#pragma unroll
    for (int a = 0; a < NB; ++a)
      atomicAdd(cnt + v[a], 1ull);
  }
}

template <int NB>
__global__ void scatter_incidences(const int32_t* __restrict__ cells, int64_t ne,
                                   unsigned long long* __restrict__ cursor, uint32_t* __restrict__ v2e)
{
  const int64_t e = blockIdx.x * static_cast<int64_t>(kT) + threadIdx.x;
  if (e >= ne)
    return;
#pragma unroll
  for (int a = 0; a < NB; ++a)
  {
    const int v = __ldg(cells + e * NB + a);
    v2e[atomicAdd(cursor + v, 1ull)] = static_cast<uint32_t>(e << 2 | a);
  }
}

// Sorted unique neighbours of v (its incident elements' vertices) in nb_out;
// returns the count, or -1 beyond kMaxDeg.
template <int NB>
__device__ int neighbours(const int32_t* __restrict__ cells, const uint32_t* __restrict__ v2e, int64_t q0,
                          int64_t q1, int32_t* nb_out)
{
  int n = 0;
  for (int64_t q = q0; q < q1; ++q)
  {
    const int64_t e = v2e[q] >> 2;
#pragma unroll
    for (int b = 0; b < NB; ++b)
    {
      const int32_t u = __ldg(cells + e * NB + b);
      int lo = 0, hi = n;
      while (lo < hi)
      {
        const int mid = (lo + hi) >> 1;
        if (nb_out[mid] < u)
          lo = mid + 1;
        else
          hi = mid;
      }
      if (lo < n && nb_out[lo] == u)
        continue;
      if (n == kMaxDeg)
        return -1;
      for (int t = n; t > lo; --t)
        nb_out[t] = nb_out[t - 1];
      nb_out[lo] = u;
      ++n;
    }
  }
  return n;
}

template <int NB>
__global__ void sort_and_degree(const int32_t* __restrict__ cells, const long long* __restrict__ v2e_ptr,
                                uint32_t* __restrict__ v2e, int64_t nv, long long* __restrict__ deg,
                                unsigned long long* __restrict__ bad)
{
  const int64_t v = blockIdx.x * static_cast<int64_t>(kT) + threadIdx.x;
  if (v >= nv)
    return;
  const int64_t q0 = v2e_ptr[v], q1 = v2e_ptr[v + 1];
  for (int64_t i = q0 + 1; i < q1; ++i)  // insertion sort: lists are short
  {
    const uint32_t x = v2e[i];
    int64_t j = i - 1;
    while (j >= q0 && v2e[j] > x)
    {
      v2e[j + 1] = v2e[j];
      --j;
    }
    v2e[j + 1] = x;
  }
  int32_t nbrs[kMaxDeg];
  const int n = neighbours<NB>(cells, v2e, q0, q1, nbrs);
  if (n < 0)
    atomicMin(bad + 2, static_cast<unsigned long long>(v));
  deg[v] = n < 0 ? 0 : n;
}

__global__ void group_widths(const long long* __restrict__ v2e_ptr, int64_t nv, long long* __restrict__ gw)
{
  const int64_t v = blockIdx.x * static_cast<int64_t>(kT) + threadIdx.x;
  const int64_t g = v / 32;
  if (g * 32 >= nv)
    return;
  int c = v < nv ? static_cast<int>(v2e_ptr[v + 1] - v2e_ptr[v]) : 0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
    c = max(c, __shfl_xor_sync(0xffffffffu, c, o));
  if ((threadIdx.x & 31) == 0)
    gw[g] = 32ll * c;
}

template <int NB>
__global__ void fill_plan(const int32_t* __restrict__ cells, const long long* __restrict__ v2e_ptr,
                          const uint32_t* __restrict__ v2e, const long long* __restrict__ nbr_ptr,
                          const long long* __restrict__ goff, int64_t nv, int32_t* __restrict__ nbr,
                          uint32_t* __restrict__ spk, uint32_t* __restrict__ spos)
{
  const int64_t v = blockIdx.x * static_cast<int64_t>(kT) + threadIdx.x;
  if (v >= nv)
    return;
  const int64_t q0 = v2e_ptr[v], q1 = v2e_ptr[v + 1];
  int32_t nbrs[kMaxDeg];
  const int n = neighbours<NB>(cells, v2e, q0, q1, nbrs);
  for (int i = 0; i < n; ++i)
    nbr[nbr_ptr[v] + i] = nbrs[i];
  const int64_t at0 = goff[v / 32] + (v % 32);
  for (int64_t q = q0; q < q1; ++q)
  {
    const uint32_t pk = v2e[q];
    const int64_t e = pk >> 2;
    uint32_t w = 0;
#pragma unroll
    for (int b = 0; b < NB; ++b)
    {
      const int32_t u = __ldg(cells + e * NB + b);
      int lo = 0, hi = n;
      while (lo < hi)
      {
        const int mid = (lo + hi) >> 1;
        if (nbrs[mid] < u)
          lo = mid + 1;
        else
          hi = mid;
      }
      w |= static_cast<uint32_t>(lo) << (8 * b);
    }
    spk[at0 + 32 * (q - q0)] = pk;
    spos[at0 + 32 * (q - q0)] = w;
  }
}

// exclusive scan of n + 1 int64 values (the last input is 0 -> total at [n])
cudaError_t scan(long long* in_out_src, long long* out, int64_t n1, cudaStream_t st)
{
  size_t bytes = 0;
  cudaError_t e = cub::DeviceScan::ExclusiveSum(nullptr, bytes, in_out_src, out, n1, st);
  if (e != cudaSuccess)
    return e;
  void* tmp = nullptr;
  if ((e = cudaMallocAsync(&tmp, bytes, st)) != cudaSuccess)
    return e;
  e = cub::DeviceScan::ExclusiveSum(tmp, bytes, in_out_src, out, n1, st);
  cudaFreeAsync(tmp, st);
  return e;
}

#define FB_TRY(x)                  \
  do                               \
  {                                \
    cudaError_t e_ = (x);          \
    if (e_ != cudaSuccess)         \
      return e_;                   \
  } while (0)

template <int NB>
cudaError_t build(int64_t ne, int64_t nv, const int32_t* cells, cudaStream_t st, PlanDevice* P, int64_t* bad_out)
{
  const int64_t ngroups = (nv + 31) / 32;
  // temporaries, and on failure the plan arrays too, are freed on every exit
  // path (an FB_TRY return included)
  struct Scratch {
    cudaStream_t st;
    PlanDevice* P;
    bool ok = false;
    unsigned long long* bad = nullptr;  // [0] bad id cell, [1] repeated-vertex cell, [2] degree vertex
    long long *cnt = nullptr, *v2e_ptr = nullptr, *deg = nullptr, *gw = nullptr;
    uint32_t* v2e = nullptr;
    ~Scratch()
    {
      for (void* q : {(void*)bad, (void*)cnt, (void*)v2e_ptr, (void*)deg, (void*)gw, (void*)v2e})
        if (q)
          cudaFreeAsync(q, st);
      if (!ok)
      {
        for (void* q : {(void*)P->goff, (void*)P->spk, (void*)P->spos, (void*)P->nbr_ptr, (void*)P->nbr})
          if (q)
            cudaFreeAsync(q, st);
        *P = PlanDevice{};
      }
      cudaStreamSynchronize(st);
    }
  } T{st, P};
  unsigned long long*& bad = T.bad;
  long long *&cnt = T.cnt, *&v2e_ptr = T.v2e_ptr, *&deg = T.deg, *&gw = T.gw;
  uint32_t*& v2e = T.v2e;
  FB_TRY(cudaMallocAsync(reinterpret_cast<void**>(&bad), 3 * sizeof(long long), st));
  FB_TRY(cudaMemsetAsync(bad, 0xff, 3 * sizeof(long long), st));
  FB_TRY(cudaMallocAsync(reinterpret_cast<void**>(&cnt), (nv + 1) * sizeof(long long), st));
  FB_TRY(cudaMemsetAsync(cnt, 0, (nv + 1) * sizeof(long long), st));
  if (ne > 0)
    validate_count<NB><<<blocks_for(ne), kT, 0, st>>>(cells, ne, nv, reinterpret_cast<unsigned long long*>(cnt),
                                                      bad);
  unsigned long long hbad[3];
  FB_TRY(cudaMemcpyAsync(hbad, bad, sizeof hbad, cudaMemcpyDeviceToHost, st));
  FB_TRY(cudaStreamSynchronize(st));
  if (hbad[0] != ~0ull || hbad[1] != ~0ull)
  {
    T.ok = true;  // nothing allocated for the plan yet
    bad_out[0] = hbad[0] != ~0ull ? static_cast<int64_t>(hbad[0]) : -1;
    bad_out[1] = hbad[1] != ~0ull ? static_cast<int64_t>(hbad[1]) : -1;
    return cudaSuccess;
  }
  FB_TRY(cudaMallocAsync(reinterpret_cast<void**>(&v2e_ptr), (nv + 1) * sizeof(long long), st));
  FB_TRY(scan(cnt, v2e_ptr, nv + 1, st));
  // cnt becomes the scatter cursor
  FB_TRY(cudaMemcpyAsync(cnt, v2e_ptr, (nv + 1) * sizeof(long long), cudaMemcpyDeviceToDevice, st));
  FB_TRY(cudaMallocAsync(reinterpret_cast<void**>(&v2e), (ne * NB > 0 ? ne * NB : 1) * sizeof(uint32_t), st));
  if (ne > 0)
    scatter_incidences<NB><<<blocks_for(ne), kT, 0, st>>>(cells, ne, reinterpret_cast<unsigned long long*>(cnt),
                                                          v2e);
  FB_TRY(cudaMallocAsync(reinterpret_cast<void**>(&deg), (nv + 1) * sizeof(long long), st));
  FB_TRY(cudaMemsetAsync(deg, 0, (nv + 1) * sizeof(long long), st));
  if (nv > 0)
    sort_and_degree<NB><<<blocks_for(nv), kT, 0, st>>>(cells, v2e_ptr, v2e, nv, deg, bad);
  FB_TRY(cudaMallocAsync(reinterpret_cast<void**>(&P->nbr_ptr), (nv + 1) * sizeof(long long), st));
  FB_TRY(scan(deg, reinterpret_cast<long long*>(P->nbr_ptr), nv + 1, st));
  FB_TRY(cudaMallocAsync(reinterpret_cast<void**>(&gw), (ngroups + 1) * sizeof(long long), st));
  FB_TRY(cudaMemsetAsync(gw, 0, (ngroups + 1) * sizeof(long long), st));
  if (nv > 0)
    group_widths<<<blocks_for(ngroups * 32), kT, 0, st>>>(v2e_ptr, nv, gw);
  FB_TRY(cudaMallocAsync(reinterpret_cast<void**>(&P->goff), (ngroups + 1) * sizeof(long long), st));
  FB_TRY(scan(gw, reinterpret_cast<long long*>(P->goff), ngroups + 1, st));
  long long totals[2];
  FB_TRY(cudaMemcpyAsync(&totals[0], P->nbr_ptr + nv, sizeof(long long), cudaMemcpyDeviceToHost, st));
  FB_TRY(cudaMemcpyAsync(&totals[1], P->goff + ngroups, sizeof(long long), cudaMemcpyDeviceToHost, st));
  FB_TRY(cudaMemcpyAsync(hbad, bad, sizeof hbad, cudaMemcpyDeviceToHost, st));
  FB_TRY(cudaStreamSynchronize(st));
  P->total_nbr = totals[0];
  P->total_sell = totals[1];
  bad_out[2] = hbad[2] != ~0ull ? static_cast<int64_t>(hbad[2]) : -1;
  if (bad_out[2] < 0)
  {
    FB_TRY(cudaMallocAsync(reinterpret_cast<void**>(&P->nbr), (totals[0] > 0 ? totals[0] : 1) * sizeof(int32_t), st));
    FB_TRY(cudaMallocAsync(reinterpret_cast<void**>(&P->spk), (totals[1] > 0 ? totals[1] : 1) * sizeof(uint32_t), st));
    FB_TRY(cudaMallocAsync(reinterpret_cast<void**>(&P->spos), (totals[1] > 0 ? totals[1] : 1) * sizeof(uint32_t), st));
    FB_TRY(cudaMemsetAsync(P->spk, 0xff, totals[1] * sizeof(uint32_t), st));
    FB_TRY(cudaMemsetAsync(P->spos, 0, totals[1] * sizeof(uint32_t), st));
    if (nv > 0)
      fill_plan<NB><<<blocks_for(nv), kT, 0, st>>>(cells, v2e_ptr, v2e, reinterpret_cast<long long*>(P->nbr_ptr),
                                                   reinterpret_cast<long long*>(P->goff), nv, P->nbr, P->spk,
                                                   P->spos);
  }
  FB_TRY(cudaGetLastError());
  FB_TRY(cudaStreamSynchronize(st));
  T.ok = true;
  launch_counter().fetch_add(nv > 0 ? 5 : 1, std::memory_order_relaxed);
  return cudaSuccess;
}

}  // namespace

cudaError_t build_plan_device(int dim, int64_t ne, int64_t nv, const int32_t* cells, cudaStream_t st,
                              PlanDevice* out, int64_t* bad)
{
  bad[0] = bad[1] = bad[2] = -1;
  return dim == 2 ? build<3>(ne, nv, cells, st, out, bad) : build<4>(ne, nv, cells, st, out, bad);
}

}  // namespace fbk
