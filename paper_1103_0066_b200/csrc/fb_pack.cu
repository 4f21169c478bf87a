// GPU pack_geometry launcher and the library launch counter.
#include "fb_launch.cuh"

namespace fbk {

std::atomic<long long>& launch_counter()
{
  static std::atomic<long long> counter{0};
  return counter;
}

std::atomic<long long>* device_setup_counters()
{
  static std::atomic<long long> counters[kMaxDevices] = {};
  return counters;
}

// GPU pack_geometry (src/geometry.cpp:312-351) = the sparse kernel's
// warp-tile pipeline with G itself as the per-slot output (OP = kPack):
// prefetched gathers, FP64 geometry with the reference's exact zero signs,
// staged coalesced / bulk-TMA stores of the slot-major PackedGeometry.
template <class S, int DIM>
cudaError_t go_pack(const LaunchArgs& a, cudaStream_t st)
{
  KParamBlob kb{};
  LaunchSpec s;
  s.op = kPack;
  s.dim = DIM;
  // 2D: per-lane stores straight from registers (one 16-byte vector per slot
  // in FP32; A/B r02 at 1M: 0.0154 -> 0.0133 ms, FP64 ties).  3D (36 / 72 B
  // per slot): staged, bulk TMA (the copy ties in FP32 and loses 3 % in FP64,
  // per-lane stores lose 1.5-2x); staging needs a 16-byte aligned destination
  s.staged = DIM == 3 && (reinterpret_cast<uintptr_t>(a.out) & 15u) == 0 ? 3 : kStDirect;
  return go_store<S, DIM, kPack, kStrict, false, false, false>(s, a, kb, st);
}

cudaError_t launch_pack(int dim, int prec, const LaunchArgs& a, cudaStream_t st)
{
  if (a.nloc <= 0)
    return cudaSuccess;
  if (prec == 0)
    return dim == 2 ? go_pack<float, 2>(a, st) : go_pack<float, 3>(a, st);
  return dim == 2 ? go_pack<double, 2>(a, st) : go_pack<double, 3>(a, st);
}

}  // namespace fbk
