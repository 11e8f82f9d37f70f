// ABI plumbing: version, thread-local last error, device properties.
#include <stdarg.h>
#include <stdio.h>

#include "gs_common.cuh"

static thread_local char g_err[512] = "";

void gs_set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

// a launch helper that could not launch (and said why with gs_set_error)
static thread_local bool g_launch_failed = false;
void gs_fail_launch() { g_launch_failed = true; }

int gs_check_launch(const char* what) {
  if (g_launch_failed) {
    g_launch_failed = false;
    (void)cudaGetLastError();
    return GS_ERR_LAUNCH;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    gs_set_error("%s: %s", what, cudaGetErrorString(e));
    return GS_ERR_LAUNCH;
  }
  return GS_OK;
}

int gs_sm_count() {
  static thread_local int dev_cached = -1;
  static thread_local int sms = 0;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  if (dev != dev_cached) {
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0)
      sms = 148;
    dev_cached = dev;
  }
  return sms;
}

extern "C" int32_t gs_abi_version(void) { return GS_ABI_VERSION; }
#ifdef GS_TRACE
// measurement builds only: 16 uint64 per CTA of the next step launches
extern "C" void gs_debug_set_trace(void* buf) {
  gs::trace_buf() = static_cast<unsigned long long*>(buf);
}
#endif
extern "C" const char* gs_last_error(void) { return g_err; }
extern "C" int32_t gs_device_sm_count(void) { return gs_sm_count(); }

#ifndef GS_BUILD_VARIANTS
#define GS_BUILD_VARIANTS 0
#endif
extern "C" int32_t gs_build_flags(void) {
  return (GS_BUILD_VARIANTS ? GS_BUILD_FLAG_VARIANTS : 0) | GS_BUILD_FLAG_TMA4;
}

extern "C" int gs_host_device_pointer(const void* host_ptr, void** dev_ptr) {
  if (!host_ptr || !dev_ptr) {
    gs_set_error("gs_host_device_pointer: null pointer");
    return GS_ERR_ARG;
  }
  void* d = nullptr;
  const cudaError_t e = cudaHostGetDevicePointer(&d, const_cast<void*>(host_ptr), 0);
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    gs_set_error("gs_host_device_pointer: not page-locked mapped host memory");
    return GS_ERR_ARG;
  }
  *dev_ptr = d;
  return GS_OK;
}
