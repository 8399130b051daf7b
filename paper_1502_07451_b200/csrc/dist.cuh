// Sharded execution of the k-way partitioner across the GPUs of one box
// (SURVEY §8(e), config 4 at 2/4/8 GPUs).
//
// Rank r owns a contiguous range of vertices at every level. Per-vertex state
// that neighbours read (part, packed refinement state, fine->coarse map) is
// REPLICATED: the kernel that produces a value stores it straight into every
// rank's copy over NVLink peer memory (Rep<T>::put), so the exchange is the
// producer's epilogue, not a separate collective. Small reductions (part
// weights, planned flows, counts, level sizes) go through an all-reduce
// kernel over the same peer memory: each rank writes its contribution into a
// slot of every peer's arena, raises a flag there (system-scope release),
// waits for all flags of its own arena (acquire), and sums the slots in rank
// order — integer only, so every rank gets bit-identical results and takes
// identical control-flow decisions.
//
// Arena = one whole cudaMalloc allocation per rank (CUDA-IPC shareable; in
// loopback mode all arenas live on one GPU). Layout:
//   [0, 64)        uint32 flags[8]   flags[q] = last epoch rank q reached
//   [64, 128)      int32 err         watchdog: a barrier timed out
//   [1024, 33792)  int64 slots[2][8][kArSlots]  (parity = epoch & 1)
//   [kArenaHeader, ...)  replicated arrays, bump-allocated identically on
//                        every rank (all ranks see the same global sizes)
#pragma once
#include <stdint.h>

constexpr int kMaxRanks = 8;
constexpr int kArSlots = 256;
constexpr size_t kArenaHeader = 64 << 10;

// Replicated array: p[r] is rank r's copy as seen from this process.
template <typename T>
struct Rep {
  T *p[kMaxRanks] = {};
  int n = 1;
  __device__ __forceinline__ void put(int64_t i, T v) const {
    p[0][i] = v;
#pragma unroll 1
    for (int r = 1; r < n; ++r) p[r][i] = v;
  }
};

struct ArSeg {
  void *in = nullptr;   // local contribution
  void *out = nullptr;  // reduced result (may alias in)
  int32_t n = 0;
  int8_t is64 = 1;      // int64 (1) or int32 (0) elements
  int8_t op = 0;        // 0 sum, 1 max, 2 min
  int8_t acc = 0;       // 1: out += reduced (op sum only)
};

struct ArArgs {
  char *arena[kMaxRanks];
  int rank = 0, P = 1;
  uint32_t epoch = 0;
  int nseg = 0;
  uint64_t timeout_ns = 30ull * 1000000000ull;
  int phase = 0;  // 0: post + wait + reduce; 1: post only; 2: reduce only (host-synchronised)
  ArSeg seg[6];
};

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint32_t *p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ uint32_t *ar_flags(char *a) { return (uint32_t *)a; }
__device__ __forceinline__ int32_t *ar_err(char *a) { return (int32_t *)(a + 64); }
__device__ __forceinline__ int64_t *ar_slots(char *a, int parity, int rank) {
  return (int64_t *)(a + 1024) + ((size_t)parity * kMaxRanks + rank) * kArSlots;
}

// One CTA. Barrier + reduction of up to kArSlots values (0 values = barrier).
__global__ void __launch_bounds__(256) ar_kernel(ArArgs A) {
  const int par = A.epoch & 1;
  int off[7];
  off[0] = 0;
  for (int s = 0; s < A.nseg; ++s) off[s + 1] = off[s] + A.seg[s].n;
  const int tot = off[A.nseg];
  if (A.phase != 2) {
    for (int i = threadIdx.x; i < tot; i += blockDim.x) {
      int s = 0;
      while (i >= off[s + 1]) ++s;
      const ArSeg &g = A.seg[s];
      const int j = i - off[s];
      const int64_t v = g.is64 ? ((const int64_t *)g.in)[j] : (int64_t)((const int32_t *)g.in)[j];
      for (int r = 0; r < A.P; ++r) ar_slots(A.arena[r], par, A.rank)[i] = v;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence_system();
      for (int r = 0; r < A.P; ++r) st_release_sys(ar_flags(A.arena[r]) + A.rank, A.epoch);
    }
    if (A.phase == 1) return;
  }
  if (A.phase == 0 && threadIdx.x < A.P) {
    const uint32_t *f = ar_flags(A.arena[A.rank]) + threadIdx.x;
    const uint64_t t0 = global_ns();
    while ((int32_t)(ld_acquire_sys(f) - A.epoch) < 0) {
      // watchdog: 30 s, or fall through at once after an earlier timeout
      if (*(volatile int32_t *)ar_err(A.arena[A.rank]) ||
          global_ns() - t0 > A.timeout_ns) {
        atomicExch(ar_err(A.arena[A.rank]), 1);
        break;
      }
      __nanosleep(64);
    }
  }
  __syncthreads();
  __threadfence_system();
  for (int i = threadIdx.x; i < tot; i += blockDim.x) {
    int s = 0;
    while (i >= off[s + 1]) ++s;
    const ArSeg &g = A.seg[s];
    const int j = i - off[s];
    int64_t v = ar_slots(A.arena[A.rank], par, 0)[i];
    for (int r = 1; r < A.P; ++r) {
      const int64_t x = ((volatile int64_t *)ar_slots(A.arena[A.rank], par, r))[i];
      v = g.op == 0 ? v + x : (g.op == 1 ? (x > v ? x : v) : (x < v ? x : v));
    }
    if (g.is64) {
      int64_t *o = (int64_t *)g.out;
      o[j] = g.acc ? o[j] + v : v;
    } else {
      int32_t *o = (int32_t *)g.out;
      o[j] = (int32_t)(g.acc ? o[j] + v : v);
    }
  }
}

// Host side of one rank's view of the group.
struct Dist {
  int rank = 0, P = 1;
  bool threads = false;  // ranks are host threads of this process on one GPU (loopback)
  char *arena[kMaxRanks] = {};
  int64_t arena_bytes = 0;
  int64_t bump = kArenaHeader;
  uint32_t epoch = 0;
  bool on() const { return P > 1; }
};
