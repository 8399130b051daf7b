// Library-wide state of the C ABI: thread-local last error, launch counter,
// version, scratch-pool configuration.
#include "common.cuh"
#include <atomic>
#include <string.h>

namespace hs {

static thread_local char g_err[1024] = "";
static std::atomic<int64_t> g_launches{0};

void set_error(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

void count_launch(int64_t k) { g_launches.fetch_add(k, std::memory_order_relaxed); }

int sm_count() {
  static int cached = 0;
  if (!cached) {
    int dev = 0, v = 148;
    if (cudaGetDevice(&dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess)
      cached = v;
    else
      cached = 148;
    // keep freed scratch in the default pool: the partitioner allocates and
    // frees per level, and a release threshold of 0 would return it to the
    // driver on every stream sync.
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  }
  return cached;
}

static __global__ void iota32_kernel(int32_t *out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int32_t)i;
}

int iota32(int32_t *out, int64_t n, cudaStream_t s) {
  if (n <= 0) return HS_OK;
  iota32_kernel<<<grid_for(n, 256), 256, 0, s>>>(out, n);
  HS_CHECK_LAUNCH();
  return HS_OK;
}

}  // namespace hs

extern "C" const char *hs_last_error(void) { return hs::g_err; }
extern "C" const char *hs_version(void) { return "hetsched_b200 0.1.0 sm_100a"; }
extern "C" int64_t hs_launch_count(void) { return hs::g_launches.load(); }
