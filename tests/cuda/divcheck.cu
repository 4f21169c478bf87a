// divcheck.cu -- GPU self-test: the engine's shared-reciprocal division
// (fb_kernels.cuh: recip_refined + div_shared) must equal __ddiv_rn bit for
// bit.  Operands are drawn from a counter-based hash in several regimes:
// realistic mesh magnitudes, full random bit patterns, and exponents at the
// fast-path guard boundaries (tiny/huge/zero/denormal/inf/nan).
#include <cstdint>

#include "fb_kernels.cuh"

namespace {

__device__ __forceinline__ uint64_t mix(uint64_t x)
{
  x ^= x >> 30;
  x *= 0xbf58476d1ce4e5b9ull;
  x ^= x >> 27;
  x *= 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

__device__ double draw(uint64_t r, int regime, int which)
{
  const uint64_t mant = r & 0x000fffffffffffffull;
  const uint64_t sign = (r >> 63) << 63;
  uint64_t e;
  switch (regime)
  {
  case 0:  // mesh-like: |x| in [2^-40, 2^8]
    e = 1023 - 40 + (r >> 52) % 48;
    break;
  case 1:  // any finite exponent
    e = 1 + (r >> 52) % 2046;
    break;
  case 2:  // guard boundaries: a and b around the 2^+-500 / 2^+-400 windows and CUDA's own limits
    e = which == 0 ? ((r >> 52) & 1 ? ((r >> 53) & 1 ? 90 + (r >> 54) % 80 : 503 + (r >> 54) % 40)
                                    : ((r >> 53) & 1 ? 1900 + (r >> 54) % 147 : 1503 + (r >> 54) % 40))
                   : ((r >> 52) & 1 ? 603 + (r >> 53) % 40 : 1403 + (r >> 53) % 40);
    break;
  default:  // specials: zeros, denormals, inf, nan mixed with normals
  {
    const int k = (r >> 52) % 8;
    e = k == 0 ? 0 : (k == 1 ? 2047 : 1023 - 20 + (r >> 55) % 40);
    if (k == 2)
      return sign ? -0.0 : 0.0;
    break;
  }
  }
  return __longlong_as_double(static_cast<long long>(sign | (e << 52) | mant));
}

__global__ void check(uint64_t n, uint64_t seed, int regime, unsigned long long* bad, double* example)
{
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
  {
    const double a = draw(mix(seed ^ (2 * i)), regime, 0);
    double b = fabs(draw(mix(seed ^ (2 * i + 1)), regime, 1));  // det > 0 in the engine
    if (regime == 3 && (i & 7) == 0)
      b = -b;
    // the engine's per-element protocol: fast quotient + guard, else __ddiv_rn
    const double y = fbk::recip_refined(b);
    bool slow = !fbk::divisor_ok(b);
    double got = fbk::div_fast<true>(a, b, y, slow);
    if (slow)
      got = __ddiv_rn(a, b);
    // ZS = false may differ from __ddiv_rn only in the sign of a zero quotient
    bool slow2 = !fbk::divisor_ok(b);
    double got2 = fbk::div_fast<false>(a, b, y, slow2);
    if (slow2)
      got2 = __ddiv_rn(a, b);
    const double want = __ddiv_rn(a, b);
    const bool same = (__double_as_longlong(got) == __double_as_longlong(want) || (got != got && want != want))
                      && (__double_as_longlong(got2) == __double_as_longlong(want) || (got2 == 0.0 && want == 0.0)
                          || (got2 != got2 && want != want));
    if (!same)
    {
      if (atomicAdd(bad, 1ull) == 0)
      {
        example[0] = a;
        example[1] = b;
        example[2] = got;
        example[3] = want;
      }
    }
  }
}

}  // namespace

extern "C" int divcheck(uint64_t n, uint64_t seed, int regime, unsigned long long* mismatches, double* example)
{
  unsigned long long* d_bad = nullptr;
  double* d_ex = nullptr;
  cudaMalloc(&d_bad, sizeof(unsigned long long));
  cudaMalloc(&d_ex, 4 * sizeof(double));
  cudaMemset(d_bad, 0, sizeof(unsigned long long));
  cudaMemset(d_ex, 0, 4 * sizeof(double));
  check<<<148 * 8, 256>>>(n, seed, regime, d_bad, d_ex);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(mismatches, d_bad, sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  cudaMemcpy(example, d_ex, 4 * sizeof(double), cudaMemcpyDeviceToHost);
  cudaFree(d_bad);
  cudaFree(d_ex);
  return e == cudaSuccess ? 0 : -1;
}
