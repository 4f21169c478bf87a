// fb_launch.cuh -- template dispatch from a runtime LaunchSpec to one kernel
// instantiation.  Each fb_kernels_<prec>_<dim>.cu instantiates one (S, DIM).
#pragma once

#include <atomic>

#include "fb_kernels.cuh"

namespace fbk {

// Library-wide kernel launch counter (exported as fb_launch_counter()).
std::atomic<long long>& launch_counter();

template <class S, int DIM, int OP, int MODE, bool SYM, bool FROM_G, bool STAGED>
cudaError_t go_sparse(const LaunchArgs& a, const KParamBlob& kb, cudaStream_t st)
{
  const KP<S, DIM, OP>& kp = *reinterpret_cast<const KP<S, DIM, OP>*>(kb.bytes);
  fb_integrate_sparse<S, DIM, OP, MODE, SYM, FROM_G, STAGED>
      <<<(unsigned)num_tiles(a.nloc), kThreads, 0, st>>>(a, kp);
  launch_counter().fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

template <class S, int DIM, int OP, int MODE, bool SYM, bool FROM_G>
cudaError_t go_store(const LaunchSpec& s, const LaunchArgs& a, const KParamBlob& kb, cudaStream_t st)
{
  return s.staged ? go_sparse<S, DIM, OP, MODE, SYM, FROM_G, true>(a, kb, st)
                  : go_sparse<S, DIM, OP, MODE, SYM, FROM_G, false>(a, kb, st);
}

template <class S, int DIM, int OP, int MODE>
cudaError_t go_mode(const LaunchSpec& s, const LaunchArgs& a, const KParamBlob& kb, cudaStream_t st)
{
  // A caller-supplied G need not be symmetric, so the G-input path never
  // takes the symmetric shortcut.
  if (s.from_g)
    return go_store<S, DIM, OP, MODE, false, true>(s, a, kb, st);
  return s.path == kSparseSym ? go_store<S, DIM, OP, MODE, true, false>(s, a, kb, st)
                              : go_store<S, DIM, OP, MODE, false, false>(s, a, kb, st);
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
