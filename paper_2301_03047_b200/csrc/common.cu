// Library plumbing behind include/glr_b200.h: thread-local error text,
// version and device probe.
#include <cstdarg>
#include <cstdio>

#include "common.cuh"

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
