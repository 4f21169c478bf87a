// fb_asm_store.cuh -- write-out of a lane's contiguous CSR run in the
// assembly kernels (fb_assemble.cu, fb_assemble_g.cu).  The runs of a warp's
// lanes are far apart, so each lane's stores are separate L2 write requests:
// scalar head up to B-byte alignment, then B-byte vector stores (32:
// STG.E.ENL2.256, one full sector per request; 16: STG.128), then a scalar
// tail.  next() yields the run's values in order.
#pragma once

#include <cstdint>


// (A/B: a streaming .cs hint on these stores changes nothing measurable.)

namespace fbk {

template <class S, int B>
__device__ __forceinline__ void st_vec(S* p, const S (&q)[B / sizeof(S)])
{
  if constexpr (B == 32 && sizeof(S) == 4)
    asm volatile("st.global.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "f"(q[0]),
                 "f"(q[1]),
                 "f"(q[2]), "f"(q[3]), "f"(q[4]), "f"(q[5]), "f"(q[6]), "f"(q[7])
                 : "memory");
  else if constexpr (B == 32)
    asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(q[0]), "d"(q[1]), "d"(q[2]),
                 "d"(q[3])
                 : "memory");
  else if constexpr (sizeof(S) == 4)
    asm volatile("st.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(q[0]), "f"(q[1]), "f"(q[2]),
                 "f"(q[3])
                 : "memory");
  else
    asm volatile("st.global.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(q[0]), "d"(q[1]) : "memory");
}

// Read-only loads under an L2 evict_last policy: element rows / G entries
// that other vertices' groups re-read later stay in L2 ahead of the
// streaming plan and CSR traffic.
#define FB_EVL_POLICY "{\n\t.reg .b64 pol;\n\tcreatepolicy.fractional.L2::evict_last.b64 pol, 1.0;\n\t"
__device__ __forceinline__ float ld_el(const float* p)
{
  float x;
  asm(FB_EVL_POLICY "ld.global.nc.L2::cache_hint.f32 %0, [%1], pol;\n\t}" : "=f"(x) : "l"(p));
  return x;
}
__device__ __forceinline__ double ld_el(const double* p)
{
  double x;
  asm(FB_EVL_POLICY "ld.global.nc.L2::cache_hint.f64 %0, [%1], pol;\n\t}" : "=d"(x) : "l"(p));
  return x;
}
__device__ __forceinline__ float4 ld_el(const float4* p)
{
  float4 q;
  asm(FB_EVL_POLICY "ld.global.nc.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], pol;\n\t}"
      : "=f"(q.x), "=f"(q.y), "=f"(q.z), "=f"(q.w)
      : "l"(p));
  return q;
}
__device__ __forceinline__ double2 ld_el(const double2* p)
{
  double2 q;
  asm(FB_EVL_POLICY "ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], pol;\n\t}" : "=d"(q.x), "=d"(q.y) : "l"(p));
  return q;
}

template <class S, int B, class F>
__device__ __forceinline__ void write_seq(S* base, int64_t len, F&& next)
{
  constexpr int W = B / static_cast<int>(sizeof(S));
  int64_t head = (W - static_cast<int64_t>((reinterpret_cast<uintptr_t>(base) / sizeof(S)) % W)) % W;
  head = head < len ? head : len;
  int64_t p = 0;
  for (; p < head; ++p)
    base[p] = next();
  for (; p + W <= len; p += W)
  {
    S q[W];
#pragma unroll
    for (int t = 0; t < W; ++t)
      q[t] = next();
    st_vec<S, B>(base + p, q);
  }
  for (; p < len; ++p)
    base[p] = next();
}


#ifndef FB_ASMG_VECST
#define FB_ASMG_VECST 1
#endif
// Write-out of a vertex's CSR row block (nc rows x deg*nc entries,
// contiguous, ci-major): entry (ci, k, cj) = acc[k] on the diagonal
// (cj == ci), +0 elsewhere, written with full-sector vector stores
// (fb_asm_store.cuh).  acc reads are the lane's own shared-memory column
// ([slot][thread]): conflict-free for any k.
template <class S, int NC, int T, bool VEC = true>
__device__ __forceinline__ void write_block(S* base, int deg, const S* acc)
{
  const int64_t len = static_cast<int64_t>(deg) * NC * NC;
  int ci = 0, k = 0, cj = 0;
  auto next = [&]() -> S
  {
    const S x = cj == ci ? acc[k * T] : S(0);
    if (++cj == NC)
    {
      cj = 0;
      if (++k == deg)
      {
        k = 0;
        ++ci;
      }
    }
    return x;
  };
  if (VEC)
    write_seq<S, 32>(base, len, next);  // A/B: 16-byte stores 0.56 -> 0.43 ms (3D-E f32)
  else
    for (int64_t p = 0; p < len; ++p)
      base[p] = next();
}

}  // namespace fbk
