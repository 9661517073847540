// tm_api.cu — error state, launch accounting and version of the C ABI.
#include <atomic>
#include <string>

#include "tm_internal.cuh"

namespace tmb {

static thread_local std::string g_last_error;
static std::atomic<long long> g_launches{0};

void set_error(const std::string &msg) { g_last_error = msg; }

int fail(int code, const std::string &msg) {
  g_last_error = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char *what) {
  g_last_error = std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
  return e == cudaErrorMemoryAllocation ? TM_E_OOM : TM_E_CUDA;
}

void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

}  // namespace tmb

extern "C" int tm_abi_version(void) { return TM_ABI_VERSION; }

extern "C" int64_t tm_kernel_launch_count(void) { return tmb::g_launches.load(); }

extern "C" const char *tm_last_error(void) { return tmb::g_last_error.c_str(); }
