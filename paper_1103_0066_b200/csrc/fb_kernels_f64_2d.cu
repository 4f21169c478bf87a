// Instantiates the double, 2D kernels (see fb_kernels.cuh).
#include "fb_launch.cuh"

namespace fbk {

cudaError_t launch_integrate_f64_2d(const LaunchSpec& s, const LaunchArgs& a,
                                       const KParamBlob& kb, cudaStream_t st)
{
  return launch_integrate_t<double, 2>(s, a, kb, st);
}

}  // namespace fbk
