// tm_api.cu — error state, launch accounting and version of the C ABI.
#include <atomic>
#include <mutex>
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

// The library's own stream-ordered memory pool per device.  Freed blocks stay
// cached (release threshold = max), so a graph rebuilt in a loop or a grown
// mining scratch costs no new physical mapping — without touching the
// process-wide default pool other libraries (torch, NCCL) allocate from.
cudaMemPool_t lib_pool(int device) {
  static std::mutex mu;
  static cudaMemPool_t pools[64] = {};
  if (device < 0 || device >= 64) return nullptr;
  std::lock_guard<std::mutex> lock(mu);
  if (!pools[device]) {
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.handleTypes = cudaMemHandleTypeNone;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = device;
    cudaMemPool_t p = nullptr;
    if (cudaMemPoolCreate(&p, &props) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    uint64_t keep = UINT64_MAX;
    cudaMemPoolSetAttribute(p, cudaMemPoolAttrReleaseThreshold, &keep);
    pools[device] = p;
  }
  return pools[device];
}

cudaError_t pool_malloc(void **p, size_t n, cudaStream_t s) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  cudaMemPool_t pool = lib_pool(dev);
  return pool ? cudaMallocFromPoolAsync(p, n, pool, s) : cudaMallocAsync(p, n, s);
}

}  // namespace tmb

extern "C" int tm_abi_version(void) { return TM_ABI_VERSION; }

extern "C" int64_t tm_kernel_launch_count(void) { return tmb::g_launches.load(); }

extern "C" const char *tm_last_error(void) { return tmb::g_last_error.c_str(); }

// Page-locked host memory for outputs the device writes with overlapped D2H
// (engine.mine's FeatureMatrix values; tm_mine pieces, tm_mine.cu).
extern "C" int tm_host_alloc(int64_t bytes, void **out) {
  if (!out || bytes < 0) return tmb::fail(TM_E_BAD_ARG, "bad argument");
  *out = nullptr;
  cudaError_t e = cudaHostAlloc(out, bytes > 0 ? (size_t)bytes : 16, cudaHostAllocPortable);
  if (e != cudaSuccess) {
    *out = nullptr;
    cudaGetLastError();
    return tmb::cuda_fail(e, "cudaHostAlloc");
  }
  return TM_OK;
}

extern "C" void tm_host_free(void *p) {
  if (p) cudaFreeHost(p);
}
