// Library-level C ABI: error reporting, version, device check.
#include <stdarg.h>

#include "common.cuh"

namespace fb {
static thread_local char g_err[1024] = "";
void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}
}  // namespace fb

extern "C" const char* fb_last_error(void) { return fb::g_err; }
extern "C" int fb_abi_version(void) { return FB_ABI_VERSION; }
extern "C" int fb_device_check(void) {
  int dev = 0;
  FB_CUDA_TRY(cudaGetDevice(&dev));
  cudaDeviceProp p;
  FB_CUDA_TRY(cudaGetDeviceProperties(&p, dev));
  if (p.major != 10 || p.minor != 0) {
    fb::set_error("libfedb200 is built for sm_100a (B200); device %d is sm_%d%d (%s)", dev, p.major, p.minor, p.name);
    return FB_UNSUPPORTED;
  }
  return FB_OK;
}
