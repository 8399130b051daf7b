// Shared helpers for the hetsched_b200 C ABI: status plumbing, launch
// accounting, stream-ordered scratch, small device utilities.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdarg.h>
#include "../../include/hetsched_b200.h"

namespace hs {

void set_error(const char *fmt, ...);
void count_launch(int64_t k = 1);

#define HS_CHECK_CUDA(expr)                                                     \
  do {                                                                          \
    cudaError_t _e = (expr);                                                    \
    if (_e != cudaSuccess) {                                                    \
      ::hs::set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr,                \
                      cudaGetErrorString(_e));                                  \
      return HS_ECUDA;                                                          \
    }                                                                           \
  } while (0)

#define HS_CHECK_LAUNCH()                                                       \
  do {                                                                          \
    ::hs::count_launch();                                                       \
    cudaError_t _e = cudaGetLastError();                                        \
    if (_e != cudaSuccess) {                                                    \
      ::hs::set_error("%s:%d launch: %s", __FILE__, __LINE__,                   \
                      cudaGetErrorString(_e));                                  \
      return HS_ECUDA;                                                          \
    }                                                                           \
  } while (0)

#define HS_REQUIRE(cond, code, ...)                                             \
  do {                                                                          \
    if (!(cond)) {                                                              \
      ::hs::set_error(__VA_ARGS__);                                             \
      return (code);                                                            \
    }                                                                           \
  } while (0)

// Stream-ordered scratch buffer that frees itself (cudaFreeAsync) on scope exit.
template <typename T>
struct Scratch {
  T *p = nullptr;
  cudaStream_t s = nullptr;
  cudaError_t alloc(size_t count, cudaStream_t stream) {
    s = stream;
    if (count == 0) count = 1;
    return cudaMallocAsync((void **)&p, count * sizeof(T), stream);
  }
  ~Scratch() {
    if (p) cudaFreeAsync(p, s);
  }
  operator T *() const { return p; }
};

inline int grid_for(int64_t work, int block, int max_blocks = 148 * 32) {
  int64_t g = (work + block - 1) / block;
  if (g < 1) g = 1;
  if (g > max_blocks) g = max_blocks;
  return (int)g;
}

#ifdef __CUDACC__
// Raise *flag when any thread of the block saw `any` (call once per block,
// by every thread, after its grid-stride loop): one store per block instead
// of one same-address atomic per offending element, which serialised the
// check on graphs where most elements offend.
__device__ __forceinline__ void block_flag(bool any, int32_t *flag) {
  if (__syncthreads_or(any) && threadIdx.x == 0) *(volatile int32_t *)flag = 1;
}
#endif

// Graph-order check shared by K7, the band order and topological_order
// (stream-ordered launch): *bad = 1 when some row's first out-neighbour (the
// lists are sorted) lies at or below the row (strict = false) / strictly
// below it (strict = true); rows equal to `skip` are ignored (-1: none).
// *bad is not cleared here.
int first_edge_below(int32_t n, int32_t skip, bool strict, const int64_t *out_ptr,
                     const int32_t *out_dst, int32_t *bad, cudaStream_t s);

// out[i] = i for i < n (stream-ordered).
int iota32(int32_t *out, int64_t n, cudaStream_t s);

// Number of SMs of the current device (cached).
int sm_count();

// ---- live kernel profiling (hs_profile_*) --------------------------------
// When enabled, Prof brackets one launch with CUDA events on its stream and
// books (launches, device ms, algorithmic bytes) under the kernel's name.
bool prof_enabled();
void prof_record(const char *name, cudaEvent_t a, cudaEvent_t b, double bytes);
struct Prof {
  const char *name;
  cudaStream_t s;
  double bytes;
  cudaEvent_t a = nullptr, b = nullptr;
  Prof(const char *n, cudaStream_t st, double by) : name(n), s(st), bytes(by) {
    if (prof_enabled()) {
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a, s);
    }
  }
  // stop(): record the end now (e.g. before a host read that determines
  // `bytes`); the booking happens at destruction
  bool stopped = false;
  void stop() {
    if (a && !stopped) cudaEventRecord(b, s);
    stopped = true;
  }
  ~Prof() {
    if (a) {
      if (!stopped) cudaEventRecord(b, s);
      prof_record(name, a, b, bytes);
    }
  }
};

}  // namespace hs
