// GPU pack_geometry launcher and the library launch counter.
#include "fb_launch.cuh"

namespace fbk {

std::atomic<long long>& launch_counter()
{
  static std::atomic<long long> counter{0};
  return counter;
}

cudaError_t launch_pack(int dim, int prec, const LaunchArgs& a, cudaStream_t st)
{
  if (a.nloc <= 0)
    return cudaSuccess;
  const unsigned grid = (unsigned)num_tiles(a.nloc);
  if (prec == 0)
  {
    if (dim == 2)
      fb_pack_geometry_kernel<float, 2><<<grid, kThreads, 0, st>>>(a);
    else
      fb_pack_geometry_kernel<float, 3><<<grid, kThreads, 0, st>>>(a);
  }
  else
  {
    if (dim == 2)
      fb_pack_geometry_kernel<double, 2><<<grid, kThreads, 0, st>>>(a);
    else
      fb_pack_geometry_kernel<double, 3><<<grid, kThreads, 0, st>>>(a);
  }
  launch_counter().fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

}  // namespace fbk
