// Library plumbing behind include/glr_b200.h: thread-local error text,
// version and device probe.
#include <cstdarg>
#include <cstdio>
#include <map>
#include <mutex>
#include <utility>

#include "common.cuh"
#include "internal.cuh"

namespace glr {

static thread_local char g_last_error[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
  va_end(ap);
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return GLR_ERR_CUDA;
  }
  return GLR_OK;
}

namespace {
std::mutex g_dev_mu;
std::map<std::pair<const void*, int>, int> g_attr_cache;  // (kernel, device) -> smem bytes set
std::map<std::pair<const void*, int>, int> g_dev_cache;   // (key, device) -> cached value
}  // namespace

int ensure_smem_attr(const void* kernel, int bytes) {
  int dev = 0;
  GLR_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(g_dev_mu);
  auto it = g_attr_cache.find({kernel, dev});
  if (it != g_attr_cache.end() && it->second >= bytes) return GLR_OK;
  GLR_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  g_attr_cache[{kernel, dev}] = bytes;
  return GLR_OK;
}

static int query_sms(void*) {
  int dev = 0, sms = kNumSMs;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
    sms = kNumSMs;
  cudaGetLastError();
  return sms;
}

int cached_per_device(const void* key, int (*init)(void* ctx), void* ctx) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    cudaGetLastError();
    dev = 0;
  }
  {
    std::lock_guard<std::mutex> lock(g_dev_mu);
    auto it = g_dev_cache.find({key, dev});
    if (it != g_dev_cache.end()) return it->second;
  }
  const int v = init(ctx);  // outside the lock (may launch occupancy queries)
  std::lock_guard<std::mutex> lock(g_dev_mu);
  g_dev_cache.emplace(std::make_pair(key, dev), v);
  return v;
}

static const char kSmsKey = 0;
int device_sms() { return cached_per_device(&kSmsKey, query_sms, nullptr); }

}  // namespace glr

extern "C" const char* glr_last_error(void) { return glr::g_last_error; }

extern "C" int glr_version(void) { return 1; }

extern "C" int glr_device_info(int* sm_count, int* cc_major, int* cc_minor) {
  int dev = 0;
  GLR_CUDA(cudaGetDevice(&dev));
  GLR_CUDA(cudaDeviceGetAttribute(sm_count, cudaDevAttrMultiProcessorCount, dev));
  GLR_CUDA(cudaDeviceGetAttribute(cc_major, cudaDevAttrComputeCapabilityMajor, dev));
  GLR_CUDA(cudaDeviceGetAttribute(cc_minor, cudaDevAttrComputeCapabilityMinor, dev));
  return GLR_OK;
}
