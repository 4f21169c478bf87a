// fb_tma.cpp -- host-side TMA descriptor encoding for the staged store.
//
// The fused kernel stages a warp tile of 32 element matrices in shared memory
// with an XOR swizzle (fb_kernels.cuh, WarpStore::unit) that is exactly the
// TMA 64-byte / 128-byte swizzle when one element matrix is one 64 / 128-byte
// row (3D Laplacian-shaped forms).  The tile then leaves shared memory with a
// single cp.async.bulk.tensor store.  The descriptor is encoded per launch
// (the output pointer changes between calls); the driver entry point is
// resolved once through the runtime, so the library does not link libcuda.
#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

#include "fb_launch.cuh"

namespace fbk {

namespace {
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encoder()
{
  static std::atomic<EncodeFn> fn{nullptr};
  static std::atomic<int> tried{0};
  EncodeFn f = fn.load(std::memory_order_acquire);
  if (f || tried.load(std::memory_order_acquire))
    return f;
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q{};
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
      q == cudaDriverEntryPointSuccess)
    f = reinterpret_cast<EncodeFn>(p);
  else
    cudaGetLastError();
  fn.store(f, std::memory_order_release);
  tried.store(1, std::memory_order_release);
  return f;
}
}  // namespace

bool encode_store_map(CUtensorMap* tm, void* out, int64_t rows, int row_scalars, int scalar_bytes, int box_rows)
{
  const int row_bytes = row_scalars * scalar_bytes;
  if (row_bytes != 64 && row_bytes != 128)
    return false;
  if ((reinterpret_cast<uintptr_t>(out) & 15) != 0 || rows <= 0 || rows > 0xffffffffLL)
    return false;
  EncodeFn f = encoder();
  if (!f)
    return false;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(row_scalars), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(row_bytes)};  // bytes, dims 1..rank-1
  if (box_rows < 1 || box_rows > 256)
    return false;
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(row_scalars), static_cast<cuuint32_t>(box_rows)};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r =
      f(tm, scalar_bytes == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, out, dims,
        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
        row_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace fbk
