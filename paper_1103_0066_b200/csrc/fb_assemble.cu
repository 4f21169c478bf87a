// fb_assemble.cu -- global CSR assembly from the element-matrix store
// (the reference stops at element matrices).
//
// Deterministic gather, no atomics.  A warp owns 32 consecutive vertices and
// one row component ci; lane l walks vertex v = 32g + l's incident elements
// in ascending element order (sliced SELL-32 lists: every lane load of the
// plan is coalesced) and adds row a + ci*nb (v's local row) of each element
// matrix, all column components, into per-(neighbour, component)
// accumulators in shared memory ([slot][thread], conflict-free).  Every CSR
// entry thus receives its contributions in ascending element order from +0
// -- bitwise the serial element loop of the oracle (oracle/fb_oracle.c
// fbo_assemble).  When the variant's element matrices are bitwise symmetric
// (the sparse-symmetric kernel paths mirror one triangle) the row is read as
// the contiguous column with the widest aligned vector loads.  Incidences are
// processed U at a time so a lane has U element rows in flight.  Vertices
// with more neighbours than fit (AsmShape::SLOTS) accumulate directly in their own
// (thread-private) rows of the output.
#include <atomic>
#include <cstdint>
#include <type_traits>

#include <cuda_runtime.h>

#include "fb_asm_store.cuh"
#include "fb_devcache.h"
#include "fb_internal.h"

namespace fbk {

std::atomic<long long>& launch_counter();

namespace {

#ifndef FB_ASM_U
#define FB_ASM_U 8
#endif
// Work split and CTA shape.  A warp owns 32 consecutive vertices, one row
// component ci and NCW of the nc column components (NCW = 1: one (ci, cj)
// block per warp, more warps in flight; NCW = nc: the whole element row per
// load, fewer plan re-reads) -- chosen per shape by measurement
// (tools/asmbench.py A/B).  A thread keeps SLOTS neighbours x NCW components
// in shared memory (<= 48 KB static per CTA); vertices with more neighbours
// accumulate in their own rows of the output.  U = incidences in flight per
// lane.
#ifndef FB_ASM_NCW2
#define FB_ASM_NCW2 2  // 2D elasticity: a warp reads the whole element row (A/B: 1 is slower)
#endif
#ifndef FB_ASM_WARPS_NCW
#define FB_ASM_WARPS_NCW 2  // warps per CTA when a warp reads several column components
#endif
#ifndef FB_ASM_NCW3D64
#define FB_ASM_NCW3D64 1  // 3D elasticity FP64
#endif
#ifndef FB_ASM_U2D
#define FB_ASM_U2D FB_ASM_U
#endif
// 2D elasticity, whole rows per warp: 4 incidences in flight (A/B r02,
// 2D-E-1M: f32 0.082 -> 0.080 ms, f64 0.135 -> 0.121 -- 104 instead of 128
// registers, 18 resident warps instead of 16; the block-diagonal read keeps
// 8: f64 0.066 -> 0.080 at 4.  16 in flight loses 1.3-2x; capping the
// registers for 12 / 16 CTAs spills and loses 2-3x)
#ifndef FB_ASM_U2E
#define FB_ASM_U2E 4
#endif
// 16 incidences in flight for the latency-bound 3D elasticity FP64 gather and
// the 3D block-diagonal reads (A/B r02: 3D-E-8M f64 4.65 -> 4.09 ms, block
// diagonal f64 0.95 -> 0.89, f32 0.59 -> 0.54; 16 everywhere loses up to 2x
// on 2D and 3D-L)
#ifndef FB_ASM_U_3E64
#define FB_ASM_U_3E64 16
#endif
#ifndef FB_ASM_U_DIAG3
#define FB_ASM_U_DIAG3 16
#endif
template <class S, int DIM, int NC>
struct AsmShape {
  static constexpr int NCW = (NC == 3 && sizeof(S) == 4) ? 3 : (NC == 2 ? FB_ASM_NCW2 : (NC == 3 ? FB_ASM_NCW3D64 : 1));
  static constexpr int WARPS = NCW == 1 ? 4 : FB_ASM_WARPS_NCW;
  static constexpr int SLOTS = NCW == 1 ? 32 : 24;
  static constexpr int U = DIM == 2 ? (NC == 2 ? FB_ASM_U2E : FB_ASM_U2D)
                           : (NC == 3 && sizeof(S) == 8 ? FB_ASM_U_3E64 : (NCW == 1 ? FB_ASM_U : 4));
  // prefetch the next chunk's plan entries (registers: 3D elasticity FP64,
  // already at the register limit, is faster without -- A/B measured)
  static constexpr bool PREF = !(NC == 3 && sizeof(S) == 8);
  // batch the slot updates of one incidence (all loads, adds, stores): faster
  // in FP32, slower in FP64 (register pressure) -- A/B measured
  static constexpr bool BATCH = sizeof(S) == 4;
  static_assert(SLOTS * NCW * 32 * WARPS * sizeof(S) <= 48 * 1024, "static smem");
};
constexpr uint32_t kPad = 0xffffffffu;

template <class S>
__device__ __forceinline__ S add_rn(S a, S b);
template <>
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
template <>
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }

// N contiguous scalars from p, whose address is a multiple of A bytes
// (A = 16, 8 or 4): the widest aligned vector loads.
#ifndef FB_ASM_EVL
#define FB_ASM_EVL 1  // A/B: 3D-E f64 4.93 -> 4.67 ms, neutral elsewhere
#endif
#ifndef FB_ASM_EVL32
#define FB_ASM_EVL32 1  // FP32 rows too (A/B: 3D-E f32 1.62 -> 1.59 ms, 3D-L 0.403 -> 0.398)
#endif
// Scalars [T0, N) of the run: at each position the widest load the
// alignment allows that still fits the tail (a 6-scalar FP32 run on an
// 8-byte boundary: 3 x 8 B; on 16 B: 16 + 8 B).
template <class S, int N, int A, int T0 = 0>
__device__ __forceinline__ void load_vec(const S* p, S (&r)[N])
{
  if constexpr (T0 < N)
  {
    constexpr int W0 = A / static_cast<int>(sizeof(S)) > 0 ? A / static_cast<int>(sizeof(S)) : 1;  // scalars per load
    constexpr int W = T0 + W0 <= N ? W0 : (sizeof(S) == 4 && W0 >= 2 && T0 + 2 <= N ? 2 : 1);
    if constexpr (W == 4)
    {
      const float4 q = FB_ASM_EVL32 ? ld_el(reinterpret_cast<const float4*>(p + T0))
                                   : __ldg(reinterpret_cast<const float4*>(p + T0));
      r[T0] = q.x;
      r[T0 + 1] = q.y;
      r[T0 + 2] = q.z;
      r[T0 + 3] = q.w;
    }
    else if constexpr (W == 2 && sizeof(S) == 8)
    {
      const double2 q = FB_ASM_EVL ? ld_el(reinterpret_cast<const double2*>(p + T0))
                                  : __ldg(reinterpret_cast<const double2*>(p + T0));
      r[T0] = q.x;
      r[T0 + 1] = q.y;
    }
    else if constexpr (W == 2)
    {
      const float2 q = __ldg(reinterpret_cast<const float2*>(p + T0));
      r[T0] = q.x;
      r[T0 + 1] = q.y;
    }
    else
      r[T0] = __ldg(p + T0);
    load_vec<S, N, A, T0 + W>(p, r);
  }
}

#ifndef FB_ASM_VECST
#define FB_ASM_VECST 1
#endif
// base[p] = acc[p*T] for p < len (a lane's own shared-memory column:
// conflict-free), with full-sector vector stores (fb_asm_store.cuh).
template <class S, int T>
__device__ __forceinline__ void write_run(S* base, int len, const S* acc)
{
  // A/B: 32-byte stores win in FP64 (2D-E 0.172 -> 0.166 ms), lose on the
  // short FP32 runs (3D-L 0.402 -> 0.415)
  constexpr int B = sizeof(S) == 8 ? 32 : 16;
  int p = 0;
  write_seq<S, B>(base, len, [&]() { return acc[(p++) * T]; });
}

__host__ __device__ constexpr int gcd_i(int a, int b) { return b == 0 ? a : gcd_i(b, a % b); }

// Row i = aa + ci*NB of an element matrix, columns j = b + cj*NB for the
// N = NB*NCW columns of components cj0 .. cj0+NCW-1 (a contiguous run).
// SYM: A(i, j) == A(j, i), so the run is read from column i, contiguous.
#ifndef FB_ASM_ROWSTART
#define FB_ASM_ROWSTART 1  // A/B: alignment from the row start alone when cj0 == 0
#endif
template <class S, int NB, int KROWS, int N, bool SYM, bool CJ0 = false>
__device__ __forceinline__ void load_row(const S* blk, int i, int cj0, S (&r)[N])
{
  if constexpr (SYM)
  {
    // the store is 16-byte aligned (host check); krows^2*s, krows*s and
    // nb*s are multiples of A, so the run starts on an A-byte boundary.
    // CJ0 (the run always starts at column 0: whole rows, or block (0, 0)):
    // only krows*s matters -- 2D elasticity FP32 rows (24 B) take 8-byte
    // loads instead of 4-byte ones, FP64 (48 B) 16-byte instead of 8 (A/B
    // r02, 2D-E-1M: f32 0.102 -> 0.081 ms, f64 0.166 -> 0.134, block
    // diagonal f64 0.083 -> 0.066; the L1 data pipe was at 84 % with 23
    // sectors per gather request.  Loading the two aligned 16-byte words that
    // cover a 24-byte FP32 row and selecting by the misalignment loses:
    // 0.081 -> 0.102)
    constexpr int A = (CJ0 && FB_ASM_ROWSTART)
                          ? gcd_i(KROWS * static_cast<int>(sizeof(S)), 16)
                          : gcd_i(gcd_i(KROWS * static_cast<int>(sizeof(S)), NB * static_cast<int>(sizeof(S))), 16);
    load_vec<S, N, A>(blk + i * KROWS + cj0 * NB, r);
  }
  else
  {
#pragma unroll
    for (int j = 0; j < N; ++j)
      r[j] = __ldg(blk + i + (cj0 * NB + j) * KROWS);
  }
}

// DIAG (elasticity, FB_ASSEMBLE_BLOCK_DIAGONAL): the caller promises every
// element matrix is block diagonal over the components with equal diagonal
// blocks (integrate_mesh output of a P1-sparse variant: SURVEY 8a row A9), so
// only block (0, 0) is read -- 1/nc^2 of the store -- and one accumulator
// per neighbour serves all nc diagonal entries of the row block; the
// off-diagonal entries are written as +0, exactly the element-order sum of
// the +0 entries the generic kernel would read.
template <class S, int DIM>
struct AsmShapeDiag : AsmShape<S, DIM, 1> {
  static constexpr int U = DIM == 3 ? FB_ASM_U_DIAG3 : FB_ASM_U2D;  // incidences in flight per lane
};
template <class S, int DIM, int NC, bool DIAG>
using AsmShapeOf = std::conditional_t<DIAG, AsmShapeDiag<S, DIM>, AsmShape<S, DIM, NC>>;

template <class S, int DIM, int NC, bool SYM, bool DIAG>
// minBlocks 1 for 2D elasticity: the register allocation it gives the FP64
// kernel at U = 4 (134 registers) runs 0.121 ms on 2D-E-1M, the
// unconstrained one (124) 0.209 ms (A/B r02); 0 = unspecified elsewhere
__global__ void __launch_bounds__(32 * AsmShapeOf<S, DIM, NC, DIAG>::WARPS, DIM == 2 && NC == 2 ? 1 : 0)
    fb_assemble_kernel(const AsmArgs a)
{
  using Sh = AsmShapeOf<S, DIM, NC, DIAG>;
  constexpr int NB = DIM + 1, KROWS = NB * NC, NK = KROWS * KROWS;
  constexpr int NCW = Sh::NCW, NWC = DIAG ? 1 : NC / NCW;  // column components per warp, warps per row
  constexpr int TPG = DIAG ? 1 : NC * NWC;                  // tasks (warps) per vertex group
  constexpr int T = 32 * Sh::WARPS;
  constexpr int SLOTS = Sh::SLOTS;
  constexpr int U = Sh::U;
  __shared__ S acc_s[SLOTS * NCW * T];
  S* acc = acc_s + threadIdx.x;
  S* vals = static_cast<S*>(a.values);
  const S* store = static_cast<const S*>(a.store);
  const int lane = threadIdx.x & 31;
  const int64_t ngroups = (a.nv + 31) / 32;
  const int64_t nwarps = ngroups * TPG;
  // task descriptors (row-block offsets of the lane's vertex, the group's
  // plan range) are prefetched one task ahead, so a task's dependent chain
  // is plan -> element rows -> adds, not offsets -> plan -> rows -> adds
  struct Desc {
    int64_t r0 = 0, r1 = 0, q0 = 0, q1 = 0;
  };
  auto load_desc = [&](int64_t w)
  {
    Desc d;
    const int64_t g = w / TPG;
    const int64_t v = g * 32 + lane;
    if (v < a.nv)
    {
      d.r0 = __ldg(a.nbr_ptr + v);
      d.r1 = __ldg(a.nbr_ptr + v + 1);
    }
    d.q0 = __ldg(a.goff + g);
    d.q1 = __ldg(a.goff + g + 1);
    return d;
  };
  const int64_t wstride = static_cast<int64_t>(gridDim.x) * (T / 32);
  int64_t w = static_cast<int64_t>(blockIdx.x) * (T / 32) + (threadIdx.x >> 5);
  Desc cur;
  if (w < nwarps)
    cur = load_desc(w);
  // plan entries of the chunk about to be processed; pk_task = the task they
  // belong to (the next task's first chunk is prefetched during the current
  // task's last chunk)
  uint32_t pk[U], ps[U];
  int64_t pk_task = -1;
  auto load_plan = [&](int64_t q, int64_t qend, uint32_t (&k)[U], uint32_t (&p)[U])
  {
#pragma unroll
    for (int u = 0; u < U; ++u)
    {
      const int64_t qu = q + 32 * u;
      k[u] = qu < qend ? __ldg(a.spk + qu) : kPad;
      p[u] = qu < qend ? __ldg(a.spos + qu) : 0u;
    }
  };
  for (; w < nwarps; w += wstride)
  {
    Desc nxt;
    if (w + wstride < nwarps)
      nxt = load_desc(w + wstride);
    const int64_t g = w / TPG;
    const int sub = static_cast<int>(w - g * TPG);
    const int ci = DIAG ? 0 : sub / NWC, cj0 = DIAG ? 0 : (sub % NWC) * NCW;
    const int64_t r0 = cur.r0;
    const int deg = static_cast<int>(cur.r1 - cur.r0);
    const int64_t q0 = cur.q0, q1 = cur.q1;
    // value (neighbour slot k, column component cj0 + c) at row + k*NC + c
    const int64_t row = r0 * NC * NC + static_cast<int64_t>(ci) * deg * NC + cj0;
    const bool in_smem = deg <= SLOTS;
    // the plan entries of chunk i+1 are loaded while chunk i's element rows
    // are gathered and added (one exposed latency per chunk, not two)
    if (pk_task != w)
      load_plan(q0 + lane, q1, pk, ps);
    // zero the accumulators while the plan entries are in flight
    if (in_smem)
      for (int k = 0; k < deg * NCW; ++k)
        acc[k * T] = S(0);
    else if (DIAG)
      for (int k = 0; k < deg * NC * NC; ++k)  // the whole row block (zeros off the diagonal)
        vals[row + k] = S(0);
    else
      for (int k = 0; k < deg; ++k)
        for (int c = 0; c < NCW; ++c)
          vals[row + k * NC + c] = S(0);
    for (int64_t q = q0 + lane; q < q1; q += 32 * U)
    {
      uint32_t npk[U], nps[U];
      int64_t npk_task = w;
      if constexpr (Sh::PREF)
      {
        if (q + 32 * U < q1)
          load_plan(q + 32 * U, q1, npk, nps);
        else if (w + wstride < nwarps)
        {
          load_plan(nxt.q0 + lane, nxt.q1, npk, nps);  // the next task's first chunk
          npk_task = w + wstride;
        }
        else
          npk_task = -1;
      }
      S r[U][NB * NCW];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (pk[u] != kPad)
        {
          const int64_t e = pk[u] >> 2;
          const int aa = static_cast<int>(pk[u] & 3u);
          load_row<S, NB, KROWS, NB * NCW, SYM, (DIAG || NCW == NC)>(store + e * NK, aa + ci * NB, cj0, r[u]);
        }
      // one incidence at a time (two incidences may share a neighbour); with
      // BATCH, the nb*NCW slots of an incidence (distinct: distinct element
      // vertices) are all loaded, added and stored as a group
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (pk[u] != kPad)
        {
          int at[NB * NCW];
#pragma unroll
          for (int b = 0; b < NB; ++b)
          {
            const int k = static_cast<int>((ps[u] >> (8 * b)) & 0xffu);
#pragma unroll
            for (int c = 0; c < NCW; ++c)
              at[b * NCW + c] = in_smem ? (k * NCW + c) * T : k * NC + c;
          }
          S* base = in_smem ? acc : vals + row;
          if constexpr (Sh::BATCH)
          {
            S cur[NB * NCW];
#pragma unroll
            for (int t = 0; t < NB * NCW; ++t)
              cur[t] = base[at[t]];
#pragma unroll
            for (int b = 0; b < NB; ++b)
#pragma unroll
              for (int c = 0; c < NCW; ++c)
                cur[b * NCW + c] = add_rn(cur[b * NCW + c], r[u][b + c * NB]);
#pragma unroll
            for (int t = 0; t < NB * NCW; ++t)
              base[at[t]] = cur[t];
          }
          else
          {
#pragma unroll
            for (int b = 0; b < NB; ++b)
#pragma unroll
              for (int c = 0; c < NCW; ++c)
                base[at[b * NCW + c]] = add_rn(base[at[b * NCW + c]], r[u][b + c * NB]);
          }
        }
      if constexpr (Sh::PREF)
      {
#pragma unroll
        for (int u = 0; u < U; ++u)
        {
          pk[u] = npk[u];
          ps[u] = nps[u];
        }
        pk_task = npk_task;
      }
      else
      {
        load_plan(q + 32 * U, q1, pk, ps);
        pk_task = q + 32 * U < q1 ? w : -1;
      }
    }
    if constexpr (DIAG)
    {
      // row blocks ci = 0 .. nc-1 of the vertex: (k, cj) = acc_k on cj == ci
      const int64_t r00 = r0 * NC * NC;
      if (in_smem)
        write_block<S, NC, T>(vals + r00, deg, acc);  // one contiguous run, full-sector stores
      else
        for (int k = 0; k < deg; ++k)  // ci = 0 accumulated in place; rows ci > 0 were zeroed
        {
          const S x = vals[r00 + k * NC];
          for (int cr = 1; cr < NC; ++cr)
            vals[r00 + static_cast<int64_t>(cr) * deg * NC + k * NC + cr] = x;
        }
    }
    else if (in_smem)
    {
      if constexpr (NCW == NC && FB_ASM_VECST)
        write_run<S, T>(vals + row, deg * NC, acc);  // the whole (v, ci) row: contiguous
      else
        for (int k = 0; k < deg; ++k)
          for (int c = 0; c < NCW; ++c)
            vals[row + k * NC + c] = acc[(k * NCW + c) * T];
    }
    cur = nxt;
  }
}

template <class S, int DIM, int NC, bool SYM, bool DIAG>
cudaError_t go(const AsmArgs& a, cudaStream_t st)
{
  using Sh = AsmShapeOf<S, DIM, NC, DIAG>;
  constexpr int T = 32 * Sh::WARPS;
  const int64_t nwarps = (a.nv + 31) / 32 * (DIAG ? 1 : NC * (NC / Sh::NCW));
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
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, fb_assemble_kernel<S, DIM, NC, SYM, DIAG>, T, 0);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        return (blocks > 0 ? blocks : 1) * (sms > 0 ? sms : 1);
      },
      device_setup_counters());
  const int64_t need = (nwarps + T / 32 - 1) / (T / 32);
  const unsigned grid = static_cast<unsigned>(need < grid_cap ? need : grid_cap);
  fb_assemble_kernel<S, DIM, NC, SYM, DIAG><<<grid, T, 0, st>>>(a);
  launch_counter().fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

template <class S, int DIM, int NC>
cudaError_t go_sym(const AsmArgs& a, cudaStream_t st)
{
  if constexpr (NC > 1)
    if (a.diag)
      return a.sym ? go<S, DIM, NC, true, true>(a, st) : go<S, DIM, NC, false, true>(a, st);
  return a.sym ? go<S, DIM, NC, true, false>(a, st) : go<S, DIM, NC, false, false>(a, st);
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
