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

// The step statistics (and the strict abort flag) into page-locked host
// memory for the asynchronous error check: one warp stores them through the
// mapped pointers, a few hundred ns in the stream instead of a copy-engine
// transfer (a D2H cudaMemcpyAsync between two small steps costs the stream
// ~15-20 us, profiles/r02/small_clouds.txt).
static __global__ void mirror_kernel(const uint32_t* __restrict__ s0, uint32_t* d0, int n0,
                                     const uint32_t* __restrict__ s1, uint32_t* d1, int n1) {
  for (int i = threadIdx.x; i < n0; i += 32) d0[i] = s0[i];
  for (int i = threadIdx.x; i < n1; i += 32) d1[i] = s1[i];
}

extern "C" int gs_mirror_to_host(const void* src0, void* dst0_host, size_t bytes0,
                                 const void* src1, void* dst1_host, size_t bytes1, void* stream) {
  if ((bytes0 && (!src0 || !dst0_host)) || (bytes1 && (!src1 || !dst1_host)) || bytes0 % 4 ||
      bytes1 % 4 || bytes0 > 4096 || bytes1 > 4096) {
    gs_set_error("gs_mirror_to_host: invalid arguments");
    return GS_ERR_ARG;
  }
  void* d0 = nullptr;
  void* d1 = nullptr;
  if (bytes0 && cudaHostGetDevicePointer(&d0, dst0_host, 0) != cudaSuccess) d0 = nullptr;
  if (bytes1 && cudaHostGetDevicePointer(&d1, dst1_host, 0) != cudaSuccess) d1 = nullptr;
  if ((bytes0 && !d0) || (bytes1 && !d1)) {
    (void)cudaGetLastError();
    gs_set_error("gs_mirror_to_host: destination is not page-locked mapped host memory");
    return GS_ERR_ARG;
  }
  mirror_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(
      static_cast<const uint32_t*>(src0), static_cast<uint32_t*>(d0), (int)(bytes0 / 4),
      static_cast<const uint32_t*>(src1), static_cast<uint32_t*>(d1), (int)(bytes1 / 4));
  return gs_check_launch("gs_mirror_to_host");
}
