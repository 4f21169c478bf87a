// fb_devcache.h -- per-device, once-per-kernel launch setup.
//
// Function attributes (the dynamic shared-memory opt-in) and occupancy belong
// to a device's context, so a kernel instantiation must be set up on EVERY
// device it is launched on, not once per process: with a device list
// (fb_integrate_mesh(..., devices = {0..7})) or one process driving several
// GPUs, a process-wide cache would launch the >48 KB-staging shapes without
// the opt-in on every device but the first.  PerDevice caches one positive
// int per device id (the persistent grid's resident CTA slots, or a grid
// cap), computed by `init` on the first launch on that device.  Host-only;
// no CUDA dependency, so the logic is unit-tested on CPU
// (tests/cpp/test_devcache.cpp).
#pragma once

#include <atomic>

namespace fbk {

constexpr int kMaxDevices = 64;

// Number of (kernel instantiation, device) setups performed so far, per
// device id (exported as fb_kernel_setups(device) for the tests).
std::atomic<long long>* device_setup_counters();

struct PerDevice {
  std::atomic<int> v[kMaxDevices] = {};

  // `init` runs with `dev` current; it may run more than once if two host
  // threads race on the first launch (both compute the same value).
  template <class F>
  int get(int dev, F&& init, std::atomic<long long>* counters)
  {
    if (dev < 0 || dev >= kMaxDevices)
      return init();
    int x = v[dev].load(std::memory_order_acquire);
    if (x == 0)
    {
      x = init();
      if (x < 1)
        x = 1;
      v[dev].store(x, std::memory_order_release);
      if (counters)
        counters[dev].fetch_add(1, std::memory_order_relaxed);
    }
    return x;
  }
};

}  // namespace fbk
