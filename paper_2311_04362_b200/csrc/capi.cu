// Process-level pieces of the C ABI: error strings, version, device check,
// launch counter.
#include <cstdlib>
#include <atomic>
#include <mutex>
#include <set>
#include <tuple>
#include <cstdarg>
#include <cstdio>

#include "itsk_common.cuh"

namespace itsk {

static thread_local char g_err[1024] = "";
static std::atomic<int64_t> g_launches{0};

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

void count_launch(int64_t k) { g_launches.fetch_add(k, std::memory_order_relaxed); }

// Function attributes take effect per device (context): the caches below
// are keyed on (device, function, attribute), so a process that solves on
// cuda:0 and then cuda:1 sets them again on the second device.
namespace {
std::mutex g_attr_mu;
std::set<std::tuple<int, const void*, int>> g_attr_done;
}  // namespace

cudaError_t func_attr_once(const void* func, cudaFuncAttribute attr, int value) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(g_attr_mu);
  const auto key = std::make_tuple(dev, func, static_cast<int>(attr));
  if (g_attr_done.count(key)) return cudaSuccess;
  e = cudaFuncSetAttribute(func, attr, value);
  if (e == cudaSuccess) g_attr_done.insert(key);
  return e;
}

cudaError_t allow_max_smem(const void* func) {
  int dev = 0, optin = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  {
    std::lock_guard<std::mutex> lock(g_attr_mu);
    if (g_attr_done.count(std::make_tuple(dev, func, -1))) return cudaSuccess;
  }
  e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaFuncAttributes fa;
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, func);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             optin - static_cast<int>(fa.sharedSizeBytes));
  if (e == cudaSuccess) {
    std::lock_guard<std::mutex> lock(g_attr_mu);
    g_attr_done.insert(std::make_tuple(dev, func, -1));
  }
  return e;
}

// The device's default memory pool gives freed blocks back to the driver at
// the next synchronisation unless a release threshold is set: the sketch's
// stream-ordered scratch would then be re-mapped on every solve (measured at
// C4: ~9 ms of host time per itsk_sketch call).  Once per device.
cudaError_t keep_async_pool() {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(g_attr_mu);
  const auto key = std::make_tuple(dev, static_cast<const void*>(nullptr), -2);
  if (g_attr_done.count(key)) return cudaSuccess;
  cudaMemPool_t pool;
  e = cudaDeviceGetDefaultMemPool(&pool, dev);
  if (e != cudaSuccess) return e;
  uint64_t keep = ~0ull;
  e = cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  if (e == cudaSuccess) g_attr_done.insert(key);
  return e;
}

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("ITSK_NO_PDL");
    return !(e && atoi(e) != 0);
  }();
  return on;
}

int num_sms() {
  static int cached = 0;
  if (cached == 0) {
    int dev = 0, v = 0;
    if (cudaGetDevice(&dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && v > 0)
      cached = v;
    else
      cached = 148;
  }
  return cached;
}

}  // namespace itsk

extern "C" const char* itsk_last_error(void) { return itsk::g_err; }

extern "C" int itsk_version(void) { return 100; }

extern "C" int64_t itsk_launch_count(void) {
  return itsk::g_launches.load(std::memory_order_relaxed);
}

extern "C" int itsk_device_check(int dev) {
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= dev) {
    itsk::set_error("no CUDA device %d", dev);
    return ITSK_ENODEV;
  }
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, dev) != cudaSuccess) {
    itsk::set_error("cudaGetDeviceProperties failed");
    return ITSK_ENODEV;
  }
  if (prop.major != 10 || prop.minor != 0) {
    itsk::set_error("device %d is sm_%d%d; this library is built for sm_100a only", dev,
                    prop.major, prop.minor);
    return ITSK_ENODEV;
  }
  return ITSK_OK;
}

// ABI check for bindings: sizes of the parameter structs as compiled here
// (tests/test_capi.py compares them with the ctypes mirrors).
extern "C" int64_t itsk_struct_size(int which) {
  switch (which) {
    case 0: return static_cast<int64_t>(sizeof(itsk_loop_params));
    case 1: return static_cast<int64_t>(sizeof(itsk_loop_result));
    case 2: return static_cast<int64_t>(sizeof(itsk_peer_params));
    default: return -1;
  }
}
