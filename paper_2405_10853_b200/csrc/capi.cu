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

// ---------------------------------------------------------------- live profiler
#include <mutex>
#include <vector>
namespace fb {
struct ProfCat {
  std::vector<cudaEvent_t> ev;
  int n = 0;
  long total = 0;  // launches seen while on, including those past the event cap
  double flops = 0.0;
};
static struct {
  bool on = false;
  int cap = 0;
  ProfCat cat[3];
  std::mutex mu;
} g_prof;

bool prof_on() { return g_prof.on; }
int prof_start(int cat, cudaStream_t st) {
  std::lock_guard<std::mutex> lk(g_prof.mu);
  ProfCat& c = g_prof.cat[cat];
  if (!g_prof.on) return -1;
  ++c.total;
  if (c.n >= g_prof.cap) return -1;
  const int i = c.n++;
  cudaEventRecord(c.ev[2 * i], st);
  return i;
}
void prof_stop(int cat, int i, cudaStream_t st, double flops) {
  if (i < 0) return;
  std::lock_guard<std::mutex> lk(g_prof.mu);
  ProfCat& c = g_prof.cat[cat];
  cudaEventRecord(c.ev[2 * i + 1], st);
  c.flops += flops;
}
}  // namespace fb

extern "C" int fb_profile_begin(int max_launches) {
  std::lock_guard<std::mutex> lk(fb::g_prof.mu);
  FB_REQUIRE(max_launches > 0 && max_launches <= 1 << 20, "bad max_launches");
  for (auto& c : fb::g_prof.cat) {
    while ((int)c.ev.size() < 2 * max_launches) {
      cudaEvent_t e;
      FB_CUDA_TRY(cudaEventCreate(&e));
      c.ev.push_back(e);
    }
    c.n = 0;
    c.total = 0;
    c.flops = 0.0;
  }
  fb::g_prof.cap = max_launches;
  fb::g_prof.on = true;
  return FB_OK;
}

extern "C" int fb_profile_end(double* out) {
  std::lock_guard<std::mutex> lk(fb::g_prof.mu);
  fb::g_prof.on = false;
  for (int k = 0; k < 3; ++k) {
    fb::ProfCat& c = fb::g_prof.cat[k];
    double ms = 0.0;
    for (int i = 0; i < c.n; ++i) {
      FB_CUDA_TRY(cudaEventSynchronize(c.ev[2 * i + 1]));
      float t = 0.f;
      FB_CUDA_TRY(cudaEventElapsedTime(&t, c.ev[2 * i], c.ev[2 * i + 1]));
      ms += t;
    }
    out[3 * k + 0] = ms;
    out[3 * k + 1] = c.n;
    out[3 * k + 2] = c.flops;
    out[9 + k] = (double)c.total;
  }
  return FB_OK;
}
