// C-ABI plumbing: thread-local error text, launch counter, version.
#include "common.cuh"

#include <atomic>
#include <string>

namespace fb {

static thread_local std::string g_err;
static std::atomic<unsigned long long> g_launches{0};

void set_error(const std::string& msg) { g_err = msg; }

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

void count_launch(unsigned n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

int check_launch(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(FB_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return FB_OK;
}

}  // namespace fb

extern "C" const char* fb_last_error(void) { return fb::g_err.c_str(); }
extern "C" int fb_abi_version(void) { return 1; }
extern "C" unsigned long long fb_launch_count(void) { return fb::g_launches.load(); }
extern "C" void fb_launch_reset(void) { fb::g_launches.store(0); }
