// fb_capi_util.h -- shared pieces of the extern "C" layer (fb_capi.cpp,
// fb_assembly.cpp): the opaque variant, error plumbing (reference exception
// texts -> fb_status + fb_error), pointer-kind detection.  Not installed.
#pragma once

#include <cstdint>
#include <cstdio>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/fembatch_b200.h"
#include "fb_internal.h"

struct fb_variant {
  int op = 0, dim = 2, nb = 3, krows = 3, ncoef = 1;
  fb_kernel_config cfg{};
  int path = fbk::kDense;
  std::string description;
  std::vector<double> k;                   // AnalyticTensor doubles as given
  fbk::KParamBlob kp{};                    // sparse block, engine precision
  std::vector<unsigned char> kdense;       // dense K, engine precision
  mutable std::mutex mu;
  mutable std::map<int, void*> kdense_dev;  // per device (dense path only)
  ~fb_variant()
  {
    for (auto& [dev, p] : kdense_dev)
    {
      int cur = 0;
      cudaGetDevice(&cur);
      cudaSetDevice(dev);
      cudaFree(p);
      cudaSetDevice(cur);
    }
  }
};

namespace fbc {

// ---------------------------------------------------------------- errors
struct Error {
  int code;
  std::string msg;
  int64_t cell;
};

[[noreturn]] inline void throw_code(int code, const std::string& msg, int64_t cell = -1)
{
  throw Error{code, msg, cell};
}

[[noreturn]] inline void invalid(const std::string& msg) { throw_code(FB_ERR_INVALID_ARGUMENT, msg); }

inline void cuda_check(cudaError_t e, const char* what)
{
  if (e != cudaSuccess)
    throw_code(FB_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

inline void fill_err(fb_error* err, int code, const std::string& msg, int64_t cell)
{
  if (!err)
    return;
  err->code = code;
  err->reserved = 0;
  err->cell = cell;
  std::snprintf(err->message, sizeof err->message, "%s", msg.c_str());
}

template <class F>
int guarded(fb_error* err, F&& f)
{
  try
  {
    f();
    fill_err(err, FB_OK, "", -1);
    return FB_OK;
  }
  catch (const Error& e)
  {
    fill_err(err, e.code, e.msg, e.cell);
    return e.code;
  }
  catch (const std::invalid_argument& e)
  {
    fill_err(err, FB_ERR_INVALID_ARGUMENT, e.what(), -1);
    return FB_ERR_INVALID_ARGUMENT;
  }
  catch (const std::out_of_range& e)
  {
    fill_err(err, FB_ERR_OUT_OF_RANGE, e.what(), -1);
    return FB_ERR_OUT_OF_RANGE;
  }
  catch (const std::bad_alloc&)
  {
    fill_err(err, FB_ERR_RUNTIME, "host allocation failed", -1);
    return FB_ERR_RUNTIME;
  }
  catch (const std::exception& e)
  {
    fill_err(err, FB_ERR_RUNTIME, e.what(), -1);
    return FB_ERR_RUNTIME;
  }
}

inline size_t scalar_size(int prec) { return prec == FB_F32 ? 4 : 8; }

inline int device_count()
{
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess)
  {
    cudaGetLastError();
    return 0;
  }
  return n;
}

// Memory kind of a pointer: -1 host (pageable or pinned), else device id.
inline int pointer_device(const void* p)
{
  if (!p)
    return -1;
  cudaPointerAttributes attr{};
  if (cudaPointerGetAttributes(&attr, p) != cudaSuccess)
  {
    cudaGetLastError();
    return -1;
  }
  if (attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged)
    return attr.device;
  return -1;
}

}  // namespace fbc
