// K7 — longest-path levels and the critical-path lower bound.
//
// Reference: sim.critical_path_lower_bound (pkg/src/hetsched/sim.py:239-247):
// best[v] = max(best[p] for p in preds, default 0.0) + min(w_cpu, w_gpu).
// max is exact and each node adds once, so any topological schedule gives
// the reference's bits. Here the schedule is level-synchronous Kahn: frontier
// i holds exactly the nodes at longest-path depth i, one persistent
// cooperative kernel walks the frontiers with a grid barrier in between.
#include "common.cuh"
#include <cub/device/device_radix_sort.cuh>

namespace {

__device__ __forceinline__ double pmax(double a, double b) { return b > a ? b : a; }
__device__ __forceinline__ double pmin(double a, double b) { return b < a ? b : a; }

struct GridBarrier {
  unsigned *count, *gen;
  __device__ void sync(unsigned nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned g0 = *(volatile unsigned *)gen;
      __threadfence();
      if (atomicAdd(count, 1u) == nblocks - 1) {
        *(volatile unsigned *)count = 0;
        __threadfence();
        atomicAdd(gen, 1u);
      } else {
        while (*(volatile unsigned *)gen == g0) __nanosleep(32);
      }
      __threadfence();
    }
    __syncthreads();
  }
};

struct LevelArgs {
  hs_dag_t g;
  int mode;
  int32_t *indeg;
  int32_t *front[3];
  int32_t *counts;    // [3]
  unsigned *bar;      // [2]
  int32_t *level;
  double *finish;
  int32_t *max_level; // [1]
  unsigned long long *cp_bits;  // [1] max finish as ordered bits (finish >= 0)
  int32_t *processed; // [1]
  // mode 3 (a given assignment): part[v] of every node, dev[p] = 1 when part
  // p runs GPU kernels (w_gpu), 0 for CPU (w_cpu)
  const int32_t *part;
  const int8_t *dev;
};

constexpr int kStage = 2048;  // frontier entries staged per block and level

__global__ void levels_kernel(LevelArgs A) {
  __shared__ int32_t s_buf[kStage];
  __shared__ int s_n, s_base;
  if (threadIdx.x == 0) s_n = 0;
  __syncthreads();
  GridBarrier bar{A.bar, A.bar + 1};
  const hs_dag_t &g = A.g;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v = tid; v < g.n; v += stride) {
    int32_t d = (int32_t)(g.in_ptr[v + 1] - g.in_ptr[v]);
    A.indeg[v] = d;
    if (d == 0) A.front[0][atomicAdd(&A.counts[0], 1)] = (int32_t)v;
  }
  bar.sync(gridDim.x);
  int lmax = -1;
  double cmax = 0.0;
  int32_t done = 0;
  for (int it = 0;; ++it) {
    const int cur = it % 3, nxt = (it + 1) % 3;
    const int32_t ncur = __ldcg(&A.counts[cur]);
    if (ncur == 0) break;
    if (tid == 0) A.counts[(it + 2) % 3] = 0;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < ncur; base += stride) {
      const int64_t i = base + threadIdx.x;
      if (i >= ncur) continue;
      const int v = __ldcg(&A.front[cur][i]);
      double reach = 0.0;
      int lv = 0;
      bool first = true;
      const int pv = (A.mode == 3 && v != g.root) ? A.part[v] : 0;
      for (int64_t j = g.in_ptr[v]; j < g.in_ptr[v + 1]; ++j) {
        int p = g.in_src[j];
        double f = __ldcg(&A.finish[p]);
        if (A.mode == 3) {
          // an input crosses when it comes from another part; the root's
          // data starts in host memory, so it crosses into GPU parts only
          const bool cross = p == g.root ? A.dev[pv] != 0 : A.part[p] != pv;
          if (cross) f = f + g.w_xfer[g.in_eid[j]];
        }
        reach = first ? f : pmax(reach, f);
        first = false;
        int lp = __ldcg(&A.level[p]) + 1;
        lv = lp > lv ? lp : lv;
      }
      double dur = A.mode == 0 ? pmin(g.w_cpu[v], g.w_gpu[v])
                   : (A.mode == 1 ? g.w_gpu[v]
                                  : (A.mode == 2 ? g.w_cpu[v] : (A.dev[pv] ? g.w_gpu[v] : g.w_cpu[v])));
      double f = reach + dur;
      __stcg(&A.finish[v], f);
      __stcg(&A.level[v], lv);
      lmax = lv > lmax ? lv : lmax;
      cmax = pmax(cmax, f);
      ++done;
      for (int64_t e = g.out_ptr[v]; e < g.out_ptr[v + 1]; ++e) {
        int s = g.out_dst[e];
        if (atomicSub(&A.indeg[s], 1) == 1) {
          // block-local staging: one global atomic per flush, not per node
          int at = atomicAdd(&s_n, 1);
          if (at < kStage) s_buf[at] = s;
          else A.front[nxt][atomicAdd(&A.counts[nxt], 1)] = s;  // overflow: direct
        }
      }
    }
    __syncthreads();
    {
      const int cnt = s_n < kStage ? s_n : kStage;
      if (threadIdx.x == 0 && cnt) s_base = atomicAdd(&A.counts[nxt], cnt);
      __syncthreads();
      for (int i = threadIdx.x; i < cnt; i += blockDim.x) A.front[nxt][s_base + i] = s_buf[i];
      __syncthreads();
      if (threadIdx.x == 0) s_n = 0;
    }
    bar.sync(gridDim.x);
  }
  if (lmax >= 0) atomicMax(A.max_level, lmax);
  if (done) {
    atomicMax(A.cp_bits, (unsigned long long)__double_as_longlong(cmax));
    atomicAdd(A.processed, done);
  }
}

}  // namespace

namespace {
int levels_impl(const hs_dag_t *g, int mode, const int32_t *part, const int8_t *dev,
                int32_t *level, double *finish, double *cp_host, int32_t *n_levels_host,
                cudaStream_t s);
}

extern "C" int hs_levels(const hs_dag_t *g, int mode, int32_t *level, double *finish,
                         double *cp_host, int32_t *n_levels_host, void *stream) {
  HS_REQUIRE(g && level && finish, HS_EINVAL, "hs_levels: null argument");
  HS_REQUIRE(mode >= 0 && mode <= 2, HS_EINVAL, "hs_levels: mode must be 0..2");
  return levels_impl(g, mode, nullptr, nullptr, level, finish, cp_host, n_levels_host,
                     (cudaStream_t)stream);
}

extern "C" int hs_assigned_makespan(const hs_dag_t *g, const int32_t *part, const int8_t *dev,
                                    int32_t k, int32_t *level, double *finish,
                                    double *makespan_host, void *stream) {
  HS_REQUIRE(g && part && dev && level && finish && makespan_host, HS_EINVAL,
             "hs_assigned_makespan: null argument");
  HS_REQUIRE(k >= 1, HS_EINVAL, "hs_assigned_makespan: k must be >= 1");
  int32_t nl = 0;
  return levels_impl(g, 3, part, dev, level, finish, makespan_host, &nl, (cudaStream_t)stream);
}

namespace {
int levels_impl(const hs_dag_t *g, int mode, const int32_t *part, const int8_t *dev,
                int32_t *level, double *finish, double *cp_host, int32_t *n_levels_host,
                cudaStream_t s) {
  const int64_t n = g->n;
  hs::Scratch<int32_t> indeg, fronts, small;
  hs::Scratch<unsigned long long> cp;
  HS_CHECK_CUDA(indeg.alloc(n, s));
  HS_CHECK_CUDA(fronts.alloc(3 * n, s));
  HS_CHECK_CUDA(small.alloc(8, s));
  HS_CHECK_CUDA(cp.alloc(1, s));
  HS_CHECK_CUDA(cudaMemsetAsync(small, 0, 8 * sizeof(int32_t), s));
  HS_CHECK_CUDA(cudaMemsetAsync(cp, 0, sizeof(unsigned long long), s));
  HS_CHECK_CUDA(cudaMemsetAsync(small.p + 5, 0xff, sizeof(int32_t), s));  // max_level = -1
  LevelArgs A;
  A.g = *g;
  A.mode = mode;
  A.indeg = indeg;
  for (int i = 0; i < 3; ++i) A.front[i] = fronts.p + i * n;
  A.counts = small.p;                    // [0..2]
  A.bar = (unsigned *)(small.p + 3);     // [3..4]
  A.max_level = small.p + 5;
  A.processed = small.p + 6;
  A.cp_bits = cp;
  A.level = level;
  A.finish = finish;
  A.part = part;
  A.dev = dev;
  const int block = 256;
  int per_sm = 0;
  HS_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, levels_kernel, block, 0));
  int grid = hs::sm_count() * (per_sm < 4 ? per_sm : 4);
  int need = (int)((n + block - 1) / block);
  if (grid > need) grid = need;
  if (grid < 1) grid = 1;
  void *args[] = {&A};
  {
    // in-CSR + pred finish/level gathers + weights + finish/level writes + out-CSR
    hs::Prof P("levels", s, 16.0 * n + 8.0 * n + 4.0 * g->m + 12.0 * g->m + 16.0 * n + 12.0 * n +
                                4.0 * g->m);
    HS_CHECK_CUDA(cudaLaunchCooperativeKernel((void *)levels_kernel, grid, block, args, 0, s));
  }
  HS_CHECK_LAUNCH();
  if (cp_host || n_levels_host) {
    int32_t h[8];
    unsigned long long cpb = 0;
    HS_CHECK_CUDA(cudaMemcpyAsync(h, small, 8 * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    HS_CHECK_CUDA(cudaMemcpyAsync(&cpb, cp, sizeof cpb, cudaMemcpyDeviceToHost, s));
    HS_CHECK_CUDA(cudaStreamSynchronize(s));
    HS_REQUIRE(h[6] == n, HS_EINVAL, "graph contains a cycle (%d of %lld nodes ordered)",
               h[6], (long long)n);
    if (n_levels_host) *n_levels_host = h[5] + 1;
    if (cp_host) {
      double c;
      memcpy(&c, &cpb, sizeof c);
      *cp_host = n ? c : 0.0;
    }
  }
  return HS_OK;
}
}  // namespace

extern "C" int hs_level_order(const hs_dag_t *g, const int32_t *level, int32_t n_levels,
                              int32_t *order, void *stream) {
  HS_REQUIRE(g && level && order, HS_EINVAL, "hs_level_order: null argument");
  cudaStream_t s = (cudaStream_t)stream;
  const int n = g->n;
  hs::Scratch<int32_t> idx, keys_out;
  HS_CHECK_CUDA(idx.alloc(n, s));
  HS_CHECK_CUDA(keys_out.alloc(n, s));
  // values = 0..n-1; a stable LSD sort by level keeps index order per level
  int32_t *ip = idx;
  int rc = hs::iota32(ip, n, s);
  if (rc != HS_OK) return rc;
  int bits = 1;
  while ((1 << bits) < n_levels && bits < 31) ++bits;
  size_t temp = 0;
  HS_CHECK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, temp, level, (int32_t *)keys_out, ip,
                                                order, n, 0, bits, s));
  hs::Scratch<char> tmp;
  HS_CHECK_CUDA(tmp.alloc(temp, s));
  HS_CHECK_CUDA(cub::DeviceRadixSort::SortPairs((void *)tmp, temp, level, (int32_t *)keys_out,
                                                ip, order, n, 0, bits, s));
  hs::count_launch(4);
  return HS_OK;
}
