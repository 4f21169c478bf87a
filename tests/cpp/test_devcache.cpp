// Per-device launch setup cache (csrc/fb_devcache.h): the kernel setup
// (shared-memory opt-in + occupancy) must run once for EVERY device id a
// kernel is launched on -- not once per process -- and never again for a
// device already set up.  Host-only; fake device ids stand in for a
// multi-GPU box.
#include <atomic>
#include <cstdio>
#include <thread>
#include <vector>

#include "fb_devcache.h"

namespace fbk {
std::atomic<long long>* device_setup_counters()
{
  static std::atomic<long long> c[kMaxDevices] = {};
  return c;
}
}  // namespace fbk

static int failures = 0;
#define CHECK(x)                                                         \
  do                                                                     \
  {                                                                      \
    if (!(x))                                                            \
    {                                                                    \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #x);           \
      ++failures;                                                        \
    }                                                                    \
  } while (0)

int main()
{
  fbk::PerDevice cache;
  int calls[fbk::kMaxDevices] = {};
  auto* counters = fbk::device_setup_counters();
  // a device list {0..7} as run_job launches it (one launch per device),
  // twice: setup happens on the first launch on each device only
  for (int round = 0; round < 2; ++round)
    for (int dev = 0; dev < 8; ++dev)
    {
      const int v = cache.get(dev, [&] { ++calls[dev]; return 100 + dev; }, counters);
      CHECK(v == 100 + dev);  // per-device value, not the first device's
    }
  for (int dev = 0; dev < 8; ++dev)
  {
    CHECK(calls[dev] == 1);
    CHECK(counters[dev].load() == 1);
  }
  CHECK(counters[8].load() == 0);
  // a non-positive setup result is stored as 1 (a launch always has a grid)
  CHECK(cache.get(9, [] { return 0; }, counters) == 1);
  CHECK(cache.get(9, [] { return 7; }, counters) == 1);
  // ids outside the table are computed every time, never cached or counted
  int out_calls = 0;
  cache.get(fbk::kMaxDevices, [&] { return ++out_calls; }, counters);
  cache.get(fbk::kMaxDevices, [&] { return ++out_calls; }, counters);
  CHECK(out_calls == 2);
  // one host thread per device (run_job's fan-out): each device set up once
  fbk::PerDevice shared;
  std::atomic<int> tcalls[fbk::kMaxDevices] = {};
  std::vector<std::thread> pool;
  for (int dev = 16; dev < 24; ++dev)
    pool.emplace_back([&, dev] {
      for (int k = 0; k < 100; ++k)
        shared.get(dev, [&] { tcalls[dev].fetch_add(1); return dev; }, nullptr);
    });
  for (auto& t : pool)
    t.join();
  for (int dev = 16; dev < 24; ++dev)
    CHECK(tcalls[dev].load() == 1);
  std::printf("%d failures\n", failures);
  return failures ? 1 : 0;
}
