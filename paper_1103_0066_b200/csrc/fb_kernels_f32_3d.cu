// Instantiates the float, 3D kernels (see fb_kernels.cuh).
#include "fb_launch.cuh"

namespace fbk {

cudaError_t launch_integrate_f32_3d(const LaunchSpec& s, const LaunchArgs& a,
                                       const KParamBlob& kb, cudaStream_t st)
{
  return launch_integrate_t<float, 3>(s, a, kb, st);
}

}  // namespace fbk
