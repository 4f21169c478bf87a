// Instantiates the double, 3D kernels (see fb_kernels.cuh).
#include "fb_launch.cuh"

namespace fbk {

cudaError_t launch_integrate_f64_3d(const LaunchSpec& s, const LaunchArgs& a,
                                       const KParamBlob& kb, cudaStream_t st)
{
  return launch_integrate_t<double, 3>(s, a, kb, st);
}

}  // namespace fbk
