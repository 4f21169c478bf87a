// fb_launch.cuh -- template dispatch from a runtime LaunchSpec to one kernel
// instantiation.  Each fb_kernels_<prec>_<dim>.cu instantiates one (S, DIM).
#pragma once

#include <atomic>

#include "fb_devcache.h"
#include "fb_kernels.cuh"

#ifndef FB_DIRECT32_AUTO
#define FB_DIRECT32_AUTO 1
#endif

namespace fbk {

// Library-wide kernel launch counter (exported as fb_launch_counter()).
std::atomic<long long>& launch_counter();

// Persistent grid: every resident CTA slot on the device, capped by the tile
// count.  The shared-memory opt-in and the occupancy query run once per
// kernel instantiation PER DEVICE (fb_devcache.h): attributes belong to the
// device context, so a device list or a multi-GPU process sets up each GPU.
template <class F>
unsigned persistent_grid(F kernel, int threads, int64_t nctas, size_t smem, PerDevice& slots,
                         int cap_per_sm = 1 << 20, bool persistent = true)
{
  int dev = 0;
  cudaGetDevice(&dev);
  const int per = slots.get(
      dev,
      [&]
      {
        int blocks = 0, sms = 0;
        cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
#ifdef FB_CARVEOUT
        // A/B: preferred shared-memory carveout (percent of the maximum); the
        // rest of the 256 KB per SM is L1 for the coordinate gathers
        cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, FB_CARVEOUT);
#endif
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, kernel, threads, smem);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        blocks = blocks < cap_per_sm ? blocks : cap_per_sm;
        return (blocks > 0 ? blocks : 1) * (sms > 0 ? sms : 1);
      },
      device_setup_counters());
#ifdef FB_NONPERSIST  // A/B: one warp tile per warp everywhere
  persistent = false;
#endif
  // non-persistent: one warp tile per warp, the hardware schedules the CTAs
  // (measured faster for 3D elasticity FP64, sparse_persistent())
  return (unsigned)(!persistent || nctas < per ? nctas : per);
}

// Tensor map of a launch's store viewed as rows of one element matrix
// (krows^2 scalars) for the TMA store of swizzled warp tiles: box = 32 rows,
// swizzle = the row size (64 / 128 bytes).  False if the driver entry point is
// unavailable or the encoding is rejected (the caller then uses the LDS/STG
// copy).
bool encode_store_map(CUtensorMap* tm, void* out, int64_t rows, int row_scalars, int scalar_bytes, int box_rows);

template <class S, int DIM, int OP, int MODE, bool SYM, bool UNI, bool FROM_G, int ST>
cudaError_t go_sparse(const LaunchArgs& a, const KParamBlob& kb, cudaStream_t st)
{
  using WS = WarpStore<S, DIM, OP, SYM>;
  const KP<S, DIM, OP>& kp = *reinterpret_cast<const KP<S, DIM, OP>*>(kb.bytes);
  CUtensorMap tm{};
  if constexpr (ST == kStTma && WS::TMA == 2)
  {
    if (!encode_store_map(&tm, a.out, a.nloc, WS::NK, (int)sizeof(S), 32 * WS::TG))
      return go_sparse<S, DIM, OP, MODE, SYM, UNI, FROM_G, kStCopy>(a, kb, st);
  }
  auto kernel = fb_integrate_sparse<S, DIM, OP, MODE, SYM, UNI, FROM_G, ST>;
  constexpr size_t smem = sparse_smem_bytes<S, DIM, OP, SYM, ST>();
  static PerDevice slots;  // one cache per kernel instantiation and device
  constexpr int threads = sparse_warps<OP>() * 32;
  const int64_t nctas = (a.nloc + threads - 1) / threads;
  kernel<<<persistent_grid(kernel, threads, nctas, smem, slots, sparse_cta_cap<DIM, OP>() * 4 / sparse_warps<OP>(),
                           sparse_persistent<S, DIM, OP>()),
           threads, smem, st>>>(a, kp, tm);
  launch_counter().fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

// Shapes whose auto store path is the direct 32-byte per-lane store.
template <class S, int DIM, int OP>
constexpr bool direct32_auto()
{
  return FB_DIRECT32_AUTO != 0 && sizeof(S) == 4 && DIM == 3 && (OP == kLaplacian || OP == kWeighted);
}

template <class S, int DIM, int OP, int MODE, bool SYM, bool UNI, bool FROM_G>
cudaError_t go_store(const LaunchSpec& s, const LaunchArgs& a, const KParamBlob& kb, cudaStream_t st)
{
  switch (s.staged)
  {
  case kStDirect:
    return go_sparse<S, DIM, OP, MODE, SYM, UNI, FROM_G, kStDirect>(a, kb, st);
  case kStCopy:
    return go_sparse<S, DIM, OP, MODE, SYM, UNI, FROM_G, kStCopy>(a, kb, st);
  case kStTma:
    // TMA wherever the staged layout has a TMA form (else identical to copy)
    if constexpr (WarpStore<S, DIM, OP, SYM>::TMA != 0)
      return go_sparse<S, DIM, OP, MODE, SYM, UNI, FROM_G, kStTma>(a, kb, st);
    else
      return go_sparse<S, DIM, OP, MODE, SYM, UNI, FROM_G, kStCopy>(a, kb, st);
  default:
    // auto: 3D Laplacian-shaped FP32 matrices (64 B = 2 sectors per element)
    // leave by per-lane 32-byte stores straight from registers -- no staging
    // (A/B r02: 3D-L-16M strict 0.79 -> 0.83, fast 0.88 -> 0.93, weighted 3D
    // 0.84 -> 0.89; FP64, the other shapes and the G-input path lose) -- when
    // the store is 32-byte aligned; else the 1D
    // bulk store of linear layouts, measured faster than the LDS/STG copy;
    // the swizzled tensor store measured slower
    if constexpr (direct32_auto<S, DIM, OP>() && !FROM_G)  // packed-G input: the copy is faster (0.96 vs 0.94)
      if ((reinterpret_cast<uintptr_t>(a.out) & 31u) == 0)
        return go_sparse<S, DIM, OP, MODE, SYM, UNI, FROM_G, kStDirect>(a, kb, st);
    if constexpr (WarpStore<S, DIM, OP, SYM>::TMA == 1)
      return go_sparse<S, DIM, OP, MODE, SYM, UNI, FROM_G, kStTma>(a, kb, st);
    else
      return go_sparse<S, DIM, OP, MODE, SYM, UNI, FROM_G, kStCopy>(a, kb, st);
  }
}

template <class S, int DIM, int OP, int MODE>
cudaError_t go_mode(const LaunchSpec& s, const LaunchArgs& a, const KParamBlob& kb, cudaStream_t st)
{
  // A caller-supplied G need not be symmetric, so the G-input path never
  // takes the symmetric shortcut.
  if (s.from_g)
    return s.path == kUniformSym ? go_store<S, DIM, OP, MODE, false, true, true>(s, a, kb, st)
                                 : go_store<S, DIM, OP, MODE, false, false, true>(s, a, kb, st);
  switch (s.path)
  {
  case kUniformSym:
    return go_store<S, DIM, OP, MODE, true, true, false>(s, a, kb, st);
  case kSparseSym:
    return go_store<S, DIM, OP, MODE, true, false, false>(s, a, kb, st);
  default:
    return go_store<S, DIM, OP, MODE, false, false, false>(s, a, kb, st);
  }
}

template <class S, int DIM, int OP>
cudaError_t go_op(const LaunchSpec& s, const LaunchArgs& a, const KParamBlob& kb, cudaStream_t st)
{
  if (s.path == kDense)
  {
    if (s.from_g)
      fb_integrate_dense<S, DIM, OP, true><<<(unsigned)num_tiles(a.nloc), kThreads, 0, st>>>(a);
    else
      fb_integrate_dense<S, DIM, OP, false><<<(unsigned)num_tiles(a.nloc), kThreads, 0, st>>>(a);
    launch_counter().fetch_add(1, std::memory_order_relaxed);
    return cudaGetLastError();
  }
  return s.mode == kFast ? go_mode<S, DIM, OP, kFast>(s, a, kb, st)
                         : go_mode<S, DIM, OP, kStrict>(s, a, kb, st);
}

template <class S, int DIM>
cudaError_t launch_integrate_t(const LaunchSpec& s, const LaunchArgs& a, const KParamBlob& kb,
                               cudaStream_t st)
{
  if (a.nloc <= 0)
    return cudaSuccess;
  switch (s.op)
  {
  case kLaplacian:
    return go_op<S, DIM, kLaplacian>(s, a, kb, st);
  case kElasticity:
    return go_op<S, DIM, kElasticity>(s, a, kb, st);
  default:
    return go_op<S, DIM, kWeighted>(s, a, kb, st);
  }
}

}  // namespace fbk
