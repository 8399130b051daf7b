// K7 — longest-path levels and the critical-path lower bound.
//
// Reference: sim.critical_path_lower_bound (pkg/src/hetsched/sim.py:239-247):
// best[v] = max(best[p] for p in preds, default 0.0) + min(w_cpu, w_gpu).
// max is exact and each node adds once, so any topological schedule gives
// the reference's bits. Here the schedule is level-synchronous Kahn: frontier
// i holds exactly the nodes at longest-path depth i (so the level is the
// frontier index), one persistent cooperative kernel walks the frontiers with
// a grid barrier in between.
//
// Pull reach, push readiness: a frontier node first pulls its predecessors'
// finish times over its in-list (all of them finished at earlier levels;
// max of (finish + crossing transfer), the same max as the dataflow kernel,
// so the same bits), then decrements each successor's pending count; the
// count reaching 0 appends it to the next frontier. Both edge loops are
// flattened across the warp's lanes (warp prefix of the degrees), so a node
// of degree 10 does not leave 22 lanes idle. The only per-edge atomic is the
// 4-byte pending decrement: the pending array (40 MB at config 4) stays in
// L2, where the former pushed 8-byte reach next to it (160 MB of 16-byte
// node states) missed L2 on most edges (ncu: 14 GB of DRAM traffic for
// 100M edges, profiles/r03_ncu_k7_frontier_relabelled.json).
#include "common.cuh"
#include <cooperative_groups.h>
#include <cub/device/device_radix_sort.cuh>

namespace {

__device__ __forceinline__ double pmin(double a, double b) { return b < a ? b : a; }

struct LevelArgs {
  hs_dag_t g;
  int mode;
  // pending predecessor count per node
  uint32_t *pend;
  int32_t *front[3];
  int32_t *counts;    // [3]
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

// warp-aggregated append of the lanes with `want` to list/count
__device__ __forceinline__ void warp_append(bool want, int32_t val, int32_t *list,
                                            int32_t *count) {
  const unsigned m = __ballot_sync(0xffffffffu, want);
  if (!m) return;
  const int lane = threadIdx.x & 31;
  int base = 0;
  if (lane == __ffs(m) - 1) base = atomicAdd(count, __popc(m));
  base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
  if (want) list[base + __popc(m & ((1u << lane) - 1))] = val;
}

constexpr int kStage = 4096;  // next-frontier entries staged per block and level

// warp-aggregated append into the block's staging buffer (one shared atomic
// per warp and step; a global counter hit by every warp serialises in L2);
// overflow goes to the global list directly
__device__ __forceinline__ void stage_append(bool want, int32_t val, int32_t *s_buf, int *s_n,
                                             int32_t *list, int32_t *count) {
  const unsigned m = __ballot_sync(0xffffffffu, want);
  if (!m) return;
  const int lane = threadIdx.x & 31;
  int base = 0;
  if (lane == __ffs(m) - 1) base = atomicAdd(s_n, __popc(m));
  base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
  const int at = base + __popc(m & ((1u << lane) - 1));
  const bool spill = want && at >= kStage;
  if (want && !spill) s_buf[at] = val;
  warp_append(spill, val, list, count);
}

__global__ void __launch_bounds__(1024) levels_kernel(LevelArgs A) {
  __shared__ int32_t s_buf[kStage];
  __shared__ int s_n, s_base;
  __shared__ unsigned long long s_reach[1024 / 32][32];  // per warp: its nodes' pulled reach
  if (threadIdx.x == 0) s_n = 0;
  auto grid = cooperative_groups::this_grid();
  const hs_dag_t &g = A.g;
  const int lane = threadIdx.x & 31;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  // warp rank interleaved across blocks: a small frontier is spread over
  // every SM instead of filling the first few blocks
  const int64_t nwarps = stride >> 5;
  const int64_t wid = (int64_t)(threadIdx.x >> 5) * gridDim.x + blockIdx.x;
  for (int64_t base = tid - lane; base < g.n; base += stride) {
    const int64_t v = base + lane;
    bool src = false;
    if (v < g.n) {
      const int32_t d = (int32_t)(g.in_ptr[v + 1] - g.in_ptr[v]);
      A.pend[v] = (uint32_t)d;
      src = d == 0;
    }
    warp_append(src, (int32_t)v, A.front[0], &A.counts[0]);
  }
  grid.sync();
  int lmax = -1;
  double cmax = 0.0;
  int32_t done = 0;
  for (int it = 0;; ++it) {
    const int cur = it % 3, nxt = (it + 1) % 3;
    const int32_t ncur = __ldcg(&A.counts[cur]);
    if (ncur == 0) break;
    if (tid == 0) A.counts[(it + 2) % 3] = 0;
    // vertices per warp: 32 on a large frontier; on a small one every warp
    // takes a few, so no warp walks a long chain of edge steps while the
    // others idle into the barrier
    const int64_t per = (ncur + nwarps - 1) / nwarps;
    int vpw = 32;
    if (per < 32) {
      vpw = 1;
      while (vpw < per) vpw <<= 1;
    }
    for (int64_t c = wid * vpw; c < ncur; c += nwarps * vpw) {
      const int64_t i = c + lane;
      int v = -1, pv = 0, deg = 0, ind = 0;
      int64_t e0 = 0, j0 = 0;
      double dur = 0.0;
      if (lane < vpw && i < ncur) {
        v = __ldcg(&A.front[cur][i]);
        pv = (A.mode == 3 && v != g.root) ? A.part[v] : 0;
        dur = A.mode == 0 ? pmin(g.w_cpu[v], g.w_gpu[v])
              : (A.mode == 1 ? g.w_gpu[v]
                 : (A.mode == 2 ? g.w_cpu[v] : (A.dev[pv] ? g.w_gpu[v] : g.w_cpu[v])));
        j0 = __ldcs(g.in_ptr + v);
        ind = (int32_t)(__ldcs(g.in_ptr + v + 1) - j0);
        e0 = __ldcs(g.out_ptr + v);
        deg = (int32_t)(__ldcs(g.out_ptr + v + 1) - e0);
      }
      constexpr int kU = 4;
      // ---- pull: reach = max over the in-list of (finish + crossing transfer)
      unsigned long long *my_reach = s_reach[threadIdx.x >> 5];
      my_reach[lane] = 0ull;  // max of non-negative doubles as ordered bits
      __syncwarp();
      {
        int incl = ind;
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        const int total = __shfl_sync(0xffffffffu, incl, 31);
        const int excl = incl - ind;
        for (int t0 = 0; t0 < total; t0 += 32 * kU) {
          int owner[kU], opv[kU];
          int64_t jj[kU];
#pragma unroll
          for (int u = 0; u < kU; ++u) {
            const int t = t0 + u * 32 + lane;
            int lo = 0;
#pragma unroll
            for (int step = 16; step; step >>= 1)
              if (__shfl_sync(0xffffffffu, excl, lo + step) <= t) lo += step;
            const long long oj = __shfl_sync(0xffffffffu, (long long)j0, lo);
            const int oex = __shfl_sync(0xffffffffu, excl, lo);
            owner[u] = lo;
            opv[u] = __shfl_sync(0xffffffffu, pv, lo);
            jj[u] = t < total ? oj + (t - oex) : -1;
          }
          int us[kU];
#pragma unroll
          for (int u = 0; u < kU; ++u) us[u] = jj[u] >= 0 ? __ldcs(g.in_src + jj[u]) : 0;
#pragma unroll
          for (int u = 0; u < kU; ++u) {
            if (jj[u] < 0) continue;
            // finished at an earlier level, written by another SM: L2, not L1
            double c = __ldcg(A.finish + us[u]);
            if (A.mode == 3) {
              // an input crosses when it comes from another part; the root's
              // data starts in host memory, so it crosses into GPU parts only
              const int pu = us[u] != g.root ? A.part[us[u]] : 0;
              const bool cross = us[u] == g.root ? A.dev[opv[u]] != 0 : pu != opv[u];
              if (cross) c = c + g.w_xfer[__ldg(g.in_eid + jj[u])];
            }
            atomicMax(&my_reach[owner[u]], (unsigned long long)__double_as_longlong(c));
          }
        }
      }
      __syncwarp();
      double f = 0.0;
      if (v >= 0) {
        f = __longlong_as_double((long long)my_reach[lane]) + dur;
        __stcg(&A.finish[v], f);
        __stcs(&A.level[v], it);
        lmax = it;
        cmax = f > cmax ? f : cmax;
        ++done;
      }
      // ---- push: one pending decrement per out-edge
      int incl = deg;
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const int total = __shfl_sync(0xffffffffu, incl, 31);
      const int excl = incl - deg;
      for (int t0 = 0; t0 < total; t0 += 32 * kU) {
        int s[kU];
        bool ready[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int t = t0 + u * 32 + lane;
          int lo = 0;
#pragma unroll
          for (int step = 16; step; step >>= 1) {
            const int probe = lo + step;
            const int pe = __shfl_sync(0xffffffffu, excl, probe);
            if (pe <= t) lo = probe;
          }
          const long long oe0 = __shfl_sync(0xffffffffu, (long long)e0, lo);
          const int oex = __shfl_sync(0xffffffffu, excl, lo);
          s[u] = 0;
          ready[u] = false;
          if (t < total) {
            const int sv = __ldcs(g.out_dst + oe0 + (t - oex));
            ready[u] = atomicSub(A.pend + sv, 1u) == 1u;
            s[u] = sv;
          }
        }
#pragma unroll
        for (int u = 0; u < kU; ++u)
          stage_append(ready[u], s[u], s_buf, &s_n, A.front[nxt], &A.counts[nxt]);
      }
    }
    __syncthreads();
    {  // flush the block's staged entries: one global atomic per block
      const int cnt = s_n < kStage ? s_n : kStage;
      if (threadIdx.x == 0 && cnt) s_base = atomicAdd(&A.counts[nxt], cnt);
      __syncthreads();
      for (int i = threadIdx.x; i < cnt; i += blockDim.x) A.front[nxt][s_base + i] = s_buf[i];
      __syncthreads();
      if (threadIdx.x == 0) s_n = 0;
    }
    grid.sync();
  }
  if (lmax >= 0) atomicMax(A.max_level, lmax);
  if (done) {
    atomicMax(A.cp_bits, (unsigned long long)__double_as_longlong(cmax));
    atomicAdd(A.processed, done);
  }
}

// ---- dataflow form for DAGs numbered in topological order --------------
// When every edge u -> v has u < v, no grid barrier is needed: CTAs take
// consecutive vertex chunks from a ticket counter and every vertex pulls its
// predecessors (in-CSR), waiting until each has published its level. A
// vertex only waits on smaller ids — in its own chunk or in chunks ticketed
// earlier to warps that are already running — so the wait always ends. Both
// outputs are their own ready flags: level -1 and finish all-ones bits (a
// NaN no arithmetic produces) until written. A predecessor's level and finish
// are polled together with relaxed loads (aligned 4- and 8-byte accesses do
// not tear), so no fence orders them. Same max/add per vertex as the
// frontier kernel, so the same bits.
constexpr int kFlowBlock = 512;

__device__ __forceinline__ int32_t ld_relaxed(const int32_t *p) {
  int32_t v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed64(const double *p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(int32_t *p, int32_t v) {
  asm volatile("st.relaxed.gpu.global.s32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed64(double *p, double v) {
  asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" :: "l"(p), "d"(v) : "memory");
}
__global__ void __launch_bounds__(kFlowBlock) levels_flow(LevelArgs A, int32_t *ticket) {
  const hs_dag_t &g = A.g;
  const int lane = threadIdx.x & 31;
  int lmax = -1;
  double cmax = 0.0;
  int32_t done = 0;
  // warp-granular tickets: 32 consecutive vertices per ticket, no CTA barrier
  for (;;) {
    int t = 0;
    if (lane == 0) t = atomicAdd(ticket, 1);
    t = __shfl_sync(0xffffffffu, t, 0);
    const int64_t v = (int64_t)t * 32 + lane;
    if ((int64_t)t * 32 >= g.n) break;
    if (v >= g.n) continue;
    const int64_t j0 = g.in_ptr[v], j1 = g.in_ptr[v + 1];
    const int pv = (A.mode == 3 && v != g.root) ? A.part[v] : 0;
    const double dur = A.mode == 0 ? pmin(g.w_cpu[v], g.w_gpu[v])
                       : (A.mode == 1 ? g.w_gpu[v]
                          : (A.mode == 2 ? g.w_cpu[v] : (A.dev[pv] ? g.w_gpu[v] : g.w_cpu[v])));
    int lev = -1;
    unsigned long long reach = 0ull;  // max of non-negative doubles as ordered bits
    constexpr int kB = 8;
    for (int64_t jb = j0; jb < j1; jb += kB) {
      int32_t u[kB], lv[kB];
      unsigned long long fb[kB];
      const int nb = (int)(j1 - jb < kB ? j1 - jb : kB);
#pragma unroll
      for (int q = 0; q < kB; ++q) u[q] = q < nb ? __ldg(g.in_src + jb + q) : 0;
      // poll: every predecessor of the batch published its level and finish
      bool ready;
      do {
        ready = true;
#pragma unroll
        for (int q = 0; q < kB; ++q) {
          if (q < nb) {
            lv[q] = ld_relaxed(A.level + u[q]);
            fb[q] = ld_relaxed64(A.finish + u[q]);
            ready = ready && lv[q] >= 0 && fb[q] != ~0ull;
          }
        }
        if (!ready) __nanosleep(32);
      } while (!ready);
#pragma unroll
      for (int q = 0; q < kB; ++q) {
        if (q < nb) {
          double c = __longlong_as_double((long long)fb[q]);
          if (A.mode == 3) {
            const int pu = u[q] != g.root ? A.part[u[q]] : 0;
            const bool cross = u[q] == g.root ? A.dev[pv] != 0 : pu != pv;
            if (cross) c = c + g.w_xfer[__ldg(g.in_eid + jb + q)];
          }
          const unsigned long long cb = (unsigned long long)__double_as_longlong(c);
          reach = cb > reach ? cb : reach;
          lev = lv[q] > lev ? lv[q] : lev;
        }
      }
    }
    const double f = __longlong_as_double((long long)reach) + dur;
    st_relaxed64(A.finish + v, f);
    st_relaxed(A.level + v, lev + 1);
    lmax = lev + 1 > lmax ? lev + 1 : lmax;
    cmax = f > cmax ? f : cmax;
    ++done;
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
  hs::Scratch<int32_t> fronts, small;
  hs::Scratch<unsigned long long> cp;
  hs::Scratch<uint32_t> pend;
  HS_CHECK_CUDA(pend.alloc(n, s));
  HS_CHECK_CUDA(fronts.alloc(3 * n, s));
  HS_CHECK_CUDA(small.alloc(8, s));
  HS_CHECK_CUDA(cp.alloc(1, s));
  HS_CHECK_CUDA(cudaMemsetAsync(small, 0, 8 * sizeof(int32_t), s));
  HS_CHECK_CUDA(cudaMemsetAsync(cp, 0, sizeof(unsigned long long), s));
  HS_CHECK_CUDA(cudaMemsetAsync(small.p + 5, 0xff, sizeof(int32_t), s));  // max_level = -1
  LevelArgs A;
  A.g = *g;
  A.mode = mode;
  A.pend = pend;
  for (int i = 0; i < 3; ++i) A.front[i] = fronts.p + i * n;
  A.counts = small.p;                    // [0..2]
  A.max_level = small.p + 5;
  A.processed = small.p + 6;
  A.cp_bits = cp;
  A.level = level;
  A.finish = finish;
  A.part = part;
  A.dev = dev;
  // one 1024-thread block per SM (block shapes 256x4/8, 512x2 measured the
  // same; the grid barrier is cooperative_groups' grid sync)
  const int block = 1024;
  int per_sm = 0;
  HS_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, levels_kernel, block, 0));
  int grid = hs::sm_count() * (per_sm < 1 ? per_sm : 1);
  int need = (int)((n + block - 1) / block);
  if (grid > need) grid = need;
  if (grid < 1) grid = 1;
  // DAG numbered in topological order: the barrier-free dataflow kernel
  {
    HS_CHECK_CUDA(cudaMemsetAsync(small.p + 7, 0, sizeof(int32_t), s));
    {
      const int rc = hs::first_edge_below((int32_t)n, -1, false, g->out_ptr, g->out_dst,
                                          small.p + 7, s);
      if (rc != HS_OK) return rc;
    }
    int32_t bad = 1;
    HS_CHECK_CUDA(cudaMemcpyAsync(&bad, small.p + 7, 4, cudaMemcpyDeviceToHost, s));
    HS_CHECK_CUDA(cudaStreamSynchronize(s));
    if (!bad && n > 0) {
      HS_CHECK_CUDA(cudaMemsetAsync(level, 0xff, n * sizeof(int32_t), s));
      HS_CHECK_CUDA(cudaMemsetAsync(finish, 0xff, n * sizeof(double), s));
      HS_CHECK_CUDA(cudaMemsetAsync(small.p + 7, 0, sizeof(int32_t), s));
      int fper = 0;
      HS_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&fper, levels_flow, kFlowBlock, 0));
      int fgrid = hs::sm_count() * (fper < 1 ? 1 : fper);
      const int64_t chunks = (n + kFlowBlock - 1) / kFlowBlock;  // CTAs worth of warps
      if (fgrid > chunks) fgrid = (int)chunks;
      // in-CSR + in_src + level/finish gathers per edge + weights + writes
      hs::Prof P("levels", s, 8.0 * n + 4.0 * g->m + 12.0 * g->m + 16.0 * n + 12.0 * n +
                                  (mode == 3 ? 16.0 * g->m : 0.0));
      levels_flow<<<fgrid, kFlowBlock, 0, s>>>(A, small.p + 7);
      HS_CHECK_LAUNCH();
      goto results;
    }
  }
  {
    void *args[] = {&A};
    // per node: in_ptr for the pending init (8) + pending init (4), frontier
    // read (4), in_ptr/out_ptr pairs (32), weights (16), finish/level writes
    // (12), frontier append (4); per edge: in_src (4) + pulled finish (8) +
    // out_dst (4) + pending read-modify-write (8); mode 3 + part (4), in_eid
    // (4) and w_xfer (8) per in-edge
    hs::Prof P("levels", s, 80.0 * n + 24.0 * g->m + (mode == 3 ? 16.0 * g->m : 0.0));
    HS_CHECK_CUDA(cudaLaunchCooperativeKernel((void *)levels_kernel, grid, block, args, 0, s));
  }
  HS_CHECK_LAUNCH();
results:
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
