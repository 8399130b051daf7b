// Device topological_order (pkg/src/hetsched/graph.py:153-172): Kahn's
// algorithm with an id min-heap — the lexicographically smallest topological
// order — bit for bit, and on a cycle the reference's CycleError member (the
// smallest id whose in-degree never reached zero). Self-loops do not count in
// the in-degrees (graph.py:157-158) and never release anything.
//
// Positions are ids in ascending order, so "smallest id" = "smallest
// position".
//
// Fast path. When every edge u -> v (self-loops aside) has v > u the order is
// the identity: after 0..i-1 are popped, i's predecessors are all popped and
// i is the smallest node left. One read per row (out-lists are sorted: a
// row is bad iff its first entry is below it) decides it; creation-order
// numbered DAGs (the reference's generator, graph.py:180-305; the tiled
// Cholesky DAG) take it.
//
// General path: one persistent CTA runs batched Kahn rounds. A round takes
// B = the b smallest ready nodes (b <= 1024, from a two-level bitmap of the
// ready set), counts for every successor w how many of its remaining
// predecessors are in B and the largest B index among them (rel[w]); w is
// released by B[0..rel[w]]. The heap pops B[0], B[1], ... in order until
// some released w is smaller than the next B element: the round keeps
// B[0..c) with c = min over released w of max(rel[w] + 1, #{B <= w}), which
// is exactly the heap's prefix (every kept pop happens before any released
// node could be the minimum). Kept nodes leave the ready set, their
// successors are decremented and the released ones enter it. Rounds are few
// on DAGs numbered close to a topological order; an arbitrary numbering
// keeps only a few nodes per round (the heap order is inherently
// sequential there).
#include "common.cuh"

namespace {

constexpr int kTopoThreads = 1024;

__global__ void iota_order(int32_t n, int32_t *order) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x)
    order[v] = (int32_t)v;
}

// in-degrees without self-loops; the initial ready bitmap (both levels)
__global__ void topo_init(hs_dag_t g, int32_t *rem, int32_t *hit, int32_t *rel, uint32_t *bm0,
                          uint32_t *bm1, int32_t *ready) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < g.n;
       v += (int64_t)gridDim.x * blockDim.x) {
    int32_t d = 0;
    for (int64_t j = g.in_ptr[v]; j < g.in_ptr[v + 1]; ++j) d += g.in_src[j] != (int32_t)v;
    rem[v] = d;
    hit[v] = 0;
    rel[v] = -1;
    if (d == 0) {
      atomicOr(bm0 + (v >> 5), 1u << (v & 31));
      atomicOr(bm1 + (v >> 10), 1u << ((v >> 5) & 31));
      atomicAdd(ready, 1);
    }
  }
}

struct TopoArgs {
  hs_dag_t g;
  int32_t *rem, *hit, *rel;
  uint32_t *bm0, *bm1;  // ready set: node bits, nonzero-word bits
  int32_t *order;
  int32_t *ready;       // [1] ready count (init), then: [0] popped, [1] rounds
};

__device__ __forceinline__ int block_exscan(int x, int *s_tmp, int *total) {
  // exclusive scan over the block (kTopoThreads = 32 warps)
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int inc = x;
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) s_tmp[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    int w = s_tmp[lane];
    int wi = w;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += y;
    }
    s_tmp[lane] = wi - w;
    if (lane == 31) *total = wi;
  }
  __syncthreads();
  const int r = s_tmp[wid] + inc - x;
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(kTopoThreads, 1) topo_rounds(TopoArgs A) {
  const hs_dag_t &g = A.g;
  const int n = g.n;
  const int W0 = (n + 31) >> 5, W1 = (W0 + 31) >> 5;
  __shared__ int32_t s_B[kTopoThreads];
  __shared__ int s_tmp[32];
  __shared__ int s_total, s_b, s_cut, s_minN, s_nrel;
  const int t = threadIdx.x;
  int ready = A.ready[0];
  int popped = 0, rounds = 0;
  int lo = 0;  // no ready node below lo
  while (ready > 0) {
    ++rounds;
    // ---- B: the b = min(ready, 1024) smallest ready nodes ----------------
    const int want = ready < kTopoThreads ? ready : kTopoThreads;
    if (t == 0) s_b = 0;
    int w1 = lo >> 10;  // level-1 word to start from
    __syncthreads();
    while (true) {
      // level-1 words [w1, w1 + 1024): one per thread; each names up to 32
      // nonzero level-0 words. Take the level-0 words in order.
      const int wi = w1 + t;
      const uint32_t m1 = wi < W1 ? A.bm1[wi] : 0u;
      // count set nodes under this level-1 word
      int cnt = 0;
      for (uint32_t m = m1; m; m &= m - 1) cnt += __popc(A.bm0[(wi << 5) + __ffs(m) - 1]);
      const int off = block_exscan(cnt, s_tmp, &s_total);
      const int have = s_b;
      if (cnt && have + off < want) {
        int o = have + off;
        for (uint32_t m = m1; m && o < want; m &= m - 1) {
          const int w0 = (wi << 5) + __ffs(m) - 1;
          for (uint32_t bits = A.bm0[w0]; bits && o < want; bits &= bits - 1)
            s_B[o++] = (w0 << 5) + __ffs(bits) - 1;
        }
      }
      __syncthreads();
      if (t == 0) s_b = have + s_total < want ? have + s_total : want;
      __syncthreads();
      if (s_b >= want || w1 + kTopoThreads >= W1) break;
      w1 += kTopoThreads;
    }
    const int b = s_b;
    // ---- count the B predecessors of every successor ----------------------
    const int v = t < b ? s_B[t] : -1;
    int64_t e0 = 0, e1 = 0;
    if (v >= 0) {
      e0 = g.out_ptr[v];
      e1 = g.out_ptr[v + 1];
      for (int64_t e = e0; e < e1; ++e) {
        const int w = g.out_dst[e];
        if (w == v) continue;
        atomicAdd(A.hit + w, 1);
        atomicMax(A.rel + w, t);
      }
    }
    if (t == 0) {
      s_cut = b;
      s_minN = INT_MAX;
      s_nrel = 0;
    }
    __syncthreads();
    // ---- the heap's prefix: cut before the first B element a released node
    // precedes ---------------------------------------------------------------
    if (v >= 0)
      for (int64_t e = e0; e < e1; ++e) {
        const int w = g.out_dst[e];
        if (w == v || A.rel[w] != t || A.hit[w] != A.rem[w]) continue;
        int lo2 = 0, hi2 = b;  // #{B <= w}: B is ascending and w is not in B
        while (lo2 < hi2) {
          const int mid = (lo2 + hi2) >> 1;
          if (s_B[mid] < w) lo2 = mid + 1; else hi2 = mid;
        }
        const int j = lo2 > t + 1 ? lo2 : t + 1;
        atomicMin(&s_cut, j);
      }
    __syncthreads();
    const int c = s_cut;
    // ---- keep B[0..c): output, leave the ready set; reset the counters ----
    if (v >= 0) {
      for (int64_t e = e0; e < e1; ++e) {
        const int w = g.out_dst[e];
        if (w == v) continue;
        A.hit[w] = 0;
        A.rel[w] = -1;
      }
      if (t < c) {
        A.order[popped + t] = v;
        atomicAnd(A.bm0 + (v >> 5), ~(1u << (v & 31)));
      }
    }
    __syncthreads();
    // level-1 bits of level-0 words that became empty (only words of kept
    // nodes can have)
    if (v >= 0 && t < c && A.bm0[v >> 5] == 0u)
      atomicAnd(A.bm1 + (v >> 10), ~(1u << ((v >> 5) & 31)));
    __syncthreads();
    // ---- successors of the kept nodes: released ones enter the ready set --
    if (v >= 0 && t < c)
      for (int64_t e = e0; e < e1; ++e) {
        const int w = g.out_dst[e];
        if (w == v) continue;
        if (atomicSub(A.rem + w, 1) == 1) {
          atomicOr(A.bm0 + (w >> 5), 1u << (w & 31));
          atomicOr(A.bm1 + (w >> 10), 1u << ((w >> 5) & 31));
          atomicMin(&s_minN, w);
          atomicAdd(&s_nrel, 1);
        }
      }
    __syncthreads();
    popped += c;
    ready += s_nrel - c;
    // the smallest ready node: B[c] if some of B stays, else past B[b-1];
    // or a released node
    int nlo = c < b ? s_B[c] : s_B[b - 1] + 1;
    if (s_minN < nlo) nlo = s_minN;
    lo = nlo;
    __syncthreads();
  }
  if (t == 0) {
    A.ready[0] = popped;
    A.ready[1] = rounds;
  }
}

__global__ void topo_stuck(int32_t n, const int32_t *rem, int32_t *first) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x)
    if (rem[v] > 0) atomicMin(first, (int32_t)v);
}

}  // namespace

extern "C" int hs_topological_order(const hs_dag_t *g, int32_t *order, int32_t *count_host,
                                    int32_t *stuck_host, int32_t *rounds_host, void *stream) {
  HS_REQUIRE(g && order && count_host && stuck_host, HS_EINVAL,
             "hs_topological_order: null argument");
  HS_REQUIRE(g->n >= 0, HS_EINVAL, "hs_topological_order: negative size");
  cudaStream_t s = (cudaStream_t)stream;
  const int32_t n = g->n;
  *stuck_host = -1;
  if (rounds_host) *rounds_host = 0;
  if (n == 0) {
    *count_host = 0;
    return HS_OK;
  }
  hs::Scratch<int32_t> flag;
  HS_CHECK_CUDA(flag.alloc(4, s));
  HS_CHECK_CUDA(cudaMemsetAsync(flag, 0, 4 * sizeof(int32_t), s));
  {
    const int rc = hs::first_edge_below(n, -1, true, g->out_ptr, g->out_dst, flag, s);
    if (rc != HS_OK) return rc;
  }
  int32_t bad = 0;
  HS_CHECK_CUDA(cudaMemcpyAsync(&bad, flag, 4, cudaMemcpyDeviceToHost, s));
  HS_CHECK_CUDA(cudaStreamSynchronize(s));
  if (!bad) {  // every edge points up: the identity
    iota_order<<<hs::grid_for(n, 256), 256, 0, s>>>(n, order);
    HS_CHECK_LAUNCH();
    *count_host = n;
    return HS_OK;
  }
  const int64_t W0 = ((int64_t)n + 31) / 32, W1 = (W0 + 31) / 32;
  hs::Scratch<int32_t> rem, hit, rel;
  hs::Scratch<uint32_t> bm0, bm1;
  HS_CHECK_CUDA(rem.alloc(n, s));
  HS_CHECK_CUDA(hit.alloc(n, s));
  HS_CHECK_CUDA(rel.alloc(n, s));
  HS_CHECK_CUDA(bm0.alloc(W0, s));
  HS_CHECK_CUDA(bm1.alloc(W1, s));
  HS_CHECK_CUDA(cudaMemsetAsync(bm0, 0, W0 * 4, s));
  HS_CHECK_CUDA(cudaMemsetAsync(bm1, 0, W1 * 4, s));
  HS_CHECK_CUDA(cudaMemsetAsync(flag, 0, 4 * sizeof(int32_t), s));
  topo_init<<<hs::grid_for(n, 256), 256, 0, s>>>(*g, rem, hit, rel, bm0, bm1, flag);
  HS_CHECK_LAUNCH();
  TopoArgs A{*g, rem, hit, rel, bm0, bm1, order, flag};
  topo_rounds<<<1, kTopoThreads, 0, s>>>(A);
  HS_CHECK_LAUNCH();
  int32_t res[2] = {0, 0};
  HS_CHECK_CUDA(cudaMemcpyAsync(res, flag, 8, cudaMemcpyDeviceToHost, s));
  HS_CHECK_CUDA(cudaStreamSynchronize(s));
  *count_host = res[0];
  if (rounds_host) *rounds_host = res[1];
  if (res[0] < n) {
    HS_CHECK_CUDA(cudaMemsetAsync(flag + 2, 0x7f, 4, s));
    topo_stuck<<<hs::grid_for(n, 256), 256, 0, s>>>(n, rem, flag + 2);
    HS_CHECK_LAUNCH();
    HS_CHECK_CUDA(cudaMemcpyAsync(stuck_host, flag + 2, 4, cudaMemcpyDeviceToHost, s));
    HS_CHECK_CUDA(cudaStreamSynchronize(s));
  }
  return HS_OK;
}
