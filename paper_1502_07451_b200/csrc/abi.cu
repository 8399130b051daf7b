// Library-wide state of the C ABI: thread-local last error, launch counter,
// version, scratch-pool configuration.
#include "common.cuh"
#include <atomic>
#include <map>
#include <mutex>
#include <string>
#include <vector>
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

static __global__ void first_edge_below_kernel(int32_t n, int32_t skip, bool strict,
                                               const int64_t *out_ptr, const int32_t *out_dst,
                                               int32_t *bad) {
  bool any = false;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = out_ptr[v], e = out_ptr[v + 1];
    if (b < e && v != skip) {
      const int32_t d = __ldg(out_dst + b);
      any |= strict ? d < v : d <= v;
    }
  }
  block_flag(any, bad);
}

int first_edge_below(int32_t n, int32_t skip, bool strict, const int64_t *out_ptr,
                     const int32_t *out_dst, int32_t *bad, cudaStream_t s) {
  if (n <= 0) return HS_OK;
  first_edge_below_kernel<<<grid_for(n, 256), 256, 0, s>>>(n, skip, strict, out_ptr, out_dst, bad);
  HS_CHECK_LAUNCH();
  return HS_OK;
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

struct ProfEntry {
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pending;
  int64_t launches = 0;
  double ms = 0, bytes = 0;
};
static std::mutex g_prof_mu;
static std::map<std::string, ProfEntry> g_prof;
static std::atomic<int> g_prof_on{0};

bool prof_enabled() { return g_prof_on.load(std::memory_order_relaxed) != 0; }

void prof_record(const char *name, cudaEvent_t a, cudaEvent_t b, double bytes) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  ProfEntry &e = g_prof[name];
  e.pending.emplace_back(a, b);
  e.launches += 1;
  e.bytes += bytes;
}

static void prof_drain() {
  for (auto &kv : g_prof) {
    for (auto &ab : kv.second.pending) {
      cudaEventSynchronize(ab.second);
      float ms = 0;
      cudaEventElapsedTime(&ms, ab.first, ab.second);
      kv.second.ms += ms;
      cudaEventDestroy(ab.first);
      cudaEventDestroy(ab.second);
    }
    kv.second.pending.clear();
  }
}

}  // namespace hs

extern "C" void hs_profile_enable(int on) { hs::g_prof_on.store(on ? 1 : 0); }

extern "C" void hs_profile_reset(void) {
  std::lock_guard<std::mutex> lk(hs::g_prof_mu);
  hs::prof_drain();
  hs::g_prof.clear();
}

extern "C" int hs_profile_report(char *buf, int len) {
  std::lock_guard<std::mutex> lk(hs::g_prof_mu);
  hs::prof_drain();
  std::string out;
  char line[256];
  for (auto &kv : hs::g_prof) {
    snprintf(line, sizeof line, "%s,%lld,%.6f,%.0f\n", kv.first.c_str(),
             (long long)kv.second.launches, kv.second.ms, kv.second.bytes);
    out += line;
  }
  if (buf && len > 0) {
    strncpy(buf, out.c_str(), (size_t)len - 1);
    buf[len - 1] = 0;
  }
  return (int)out.size();
}

extern "C" const char *hs_last_error(void) { return hs::g_err; }
extern "C" const char *hs_version(void) { return "hetsched_b200 0.1.0 sm_100a"; }
extern "C" int64_t hs_launch_count(void) { return hs::g_launches.load(); }
