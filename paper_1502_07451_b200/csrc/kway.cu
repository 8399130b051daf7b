// K1/K3/K4/K5/K6 — multilevel k-way partitioning of the weighted task DAG.
//
// The paper hands its DAG to METIS; the reference ships
// a 2-way FM heuristic instead (partition.py:137-295) and lists k > 2 as a
// non-goal. This file is the B200-native METIS role for graphs far beyond
// FM's O(n^2) reach:
//   K1 symmetrize  DAG (in+out CSR) -> undirected kernel graph (root dropped,
//                  the graph emit_metis exports, graphio.py:285-304)
//   K3 matching    heavy-edge matching by locally-dominant edges: every
//                  unmatched vertex points at its best unmatched neighbour
//                  (weight, then a symmetric per-round hash, then id); mutual
//                  pointers match. A few rounds per level.
//   K4 contraction coarse ids by a scan over pair leaders; coarse adjacency
//                  = union of the pair's lists mapped through cmap, self
//                  loops dropped, parallel edges merged in a per-vertex
//                  shared-memory hash table (warp, CTA or global-memory
//                  table by list length), written into padded slots so one
//                  pass suffices.
//   K5 initial     many randomized BFS-order streaming (LDG) k-way starts on
//                  the coarsest graph, one warp each, plus greedy refinement;
//                  best (feasible, cut) wins.
//   K6 refinement  per level on the way up: parallel label-propagation
//                  moves with a Jet-style afterburner (a move survives only
//                  if it still gains assuming every higher-priority
//                  neighbouring move happened), then deterministic
//                  hash-thinned rebalancing if a part leaves its bound.
// Every reduction is integer and every tie breaks on ids/hashes, so the
// result is a pure function of (graph, k, targets, tol, seed) even though
// adjacency order inside coarse lists is not fixed.
//
// Balance (SURVEY App. B k-way generalisation of partition.py:72):
// |w_p / total - t_p| <= tol for every part p.
#include "common.cuh"
#include <cub/device/device_scan.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>
#include <cub/device/device_reduce.cuh>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_segmented_sort.cuh>
#include <vector>
#include <algorithm>
#include <cuda_profiler_api.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;
#include <mutex>
#include <condition_variable>
#include <chrono>
#include <memory>
#include "dist.cuh"


namespace {

constexpr int kMaxParts = 64;
using part_t = int8_t;  // part ids (k <= 64) as bytes: 4x less gather traffic

struct G {
  int32_t n = 0;
  int64_t cap = 0;  // adjacency slots (padded)
  int64_t nnz = 0;  // live adjacency entries
  const int32_t *twin = nullptr;  // reverse-entry positions (finest level only)
  int64_t *xbeg;
  int32_t *deg;
  int32_t *adj;
  int32_t *wgt;
  int32_t *vw;
  int32_t v0 = 0;  // global id of local vertex 0 (a rank's range when sharded)
  // Uniform edge weights (every entry == wconst; METIS's adjwgt = NULL): no
  // weight array is read or written on this level. 0: per-entry weights.
  int32_t wconst = 0;
  __device__ __forceinline__ int ew(int64_t j) const { return wconst ? wconst : __ldg(wgt + j); }
};

// L2 residency of the connectivity cache. Its rows (80 MB on config 4) are
// re-read and updated every pass, while the adjacency and state streams of the
// same pass (GBs) would evict them: cache-row accesses carry an evict_last
// policy, one-touch adjacency gathers evict_first (PTX cache hints).
__device__ __forceinline__ uint64_t l2_keep() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint2 ld_keep2(const void *ptr, uint64_t pol) {
  uint2 r;
  asm volatile("ld.global.nc.L2::cache_hint.v2.u32 {%0, %1}, [%2], %3;"
               : "=r"(r.x), "=r"(r.y) : "l"(ptr), "l"(pol));
  return r;
}
__device__ __forceinline__ uint4 ld_keep4(const void *ptr, uint64_t pol) {
  uint4 r;
  asm volatile("ld.global.nc.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(ptr), "l"(pol));
  return r;
}
__device__ __forceinline__ void st_keep2(void *ptr, unsigned long long v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.u64 [%0], %1, %2;" :: "l"(ptr), "l"(v), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void red_keep(unsigned long long *ptr, unsigned long long v,
                                         uint64_t pol) {
  asm volatile("red.global.add.L2::cache_hint.u64 [%0], %1, %2;" :: "l"(ptr), "l"(v), "l"(pol)
               : "memory");
}
__device__ __forceinline__ int32_t ld_once(const int32_t *ptr) {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  int32_t r;
  asm volatile("ld.global.nc.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(r) : "l"(ptr), "l"(pol));
  return r;
}

// Connectivity (gain) cache: row v holds kc counters of cw bytes (1, 2 or 4;
// the host picks the narrowest width that cannot overflow: every counter is at
// most v's weighted degree). Narrow rows keep the cache L2-resident.
struct Conn {
  uint8_t *p = nullptr;
  int kc = 0, cw = 4;
  __device__ __forceinline__ void set(int64_t v, int q, int val) const {
    uint8_t *a = p + (v * kc + q) * cw;
    if (cw == 1) *a = (uint8_t)val;
    else if (cw == 2) *reinterpret_cast<uint16_t *>(a) = (uint16_t)val;
    else *reinterpret_cast<int32_t *>(a) = val;
  }
  // exact update for one edge of weight w whose far end moved own -> dest:
  // word-granular atomics (no carry/borrow can cross a counter: counters stay
  // in [0, weighted degree]); one atomic when both counters share a word
  __device__ __forceinline__ void move(int64_t u, int own, int dest, int w) const {
    const int64_t row = u * kc * cw;
    if (cw == 4) {
      atomicAdd(reinterpret_cast<int32_t *>(p + row) + own, -w);
      atomicAdd(reinterpret_cast<int32_t *>(p + row) + dest, w);
      return;
    }
    if (kc * cw == 8) {  // 8-byte rows: one 64-bit atomic for both counters (no
                         // borrow/carry can cross a counter, as below)
      const unsigned long long delta = ((unsigned long long)(unsigned)w << (8 * cw * dest)) -
                                       ((unsigned long long)(unsigned)w << (8 * cw * own));
      red_keep(reinterpret_cast<unsigned long long *>(p + row), delta, l2_keep());
      return;
    }
    const int64_t bo = row + own * cw, bd = row + dest * cw;
    const unsigned so = (unsigned)(bo & 3) * 8u, sd = (unsigned)(bd & 3) * 8u;
    unsigned *wo = reinterpret_cast<unsigned *>(p + (bo & ~3ll));
    unsigned *wd = reinterpret_cast<unsigned *>(p + (bd & ~3ll));
    const unsigned dn = 0u - ((unsigned)w << so), up = (unsigned)w << sd;
    if (wo == wd) {
      atomicAdd(wo, dn + up);
    } else {
      atomicAdd(wo, dn);
      atomicAdd(wd, up);
    }
  }
};

// KC counters of CW bytes of row v (KC * CW is 8, 16, 32 or 64 bytes)
template <int KC, int CW>
__device__ __forceinline__ void conn_row(const uint8_t *p, int64_t v, int (&c)[KC]) {
  constexpr int WORDS = KC * CW / 4;
  uint32_t w[WORDS];
  const uint8_t *row = p + v * KC * CW;
  if constexpr (WORDS == 2) {
    const uint2 x = ld_keep2(row, l2_keep());
    w[0] = x.x; w[1] = x.y;
  } else {
#pragma unroll
    for (int i = 0; i < WORDS / 4; ++i) {
      const uint4 x = __ldg(reinterpret_cast<const uint4 *>(row) + i);
      w[4 * i] = x.x; w[4 * i + 1] = x.y; w[4 * i + 2] = x.z; w[4 * i + 3] = x.w;
    }
  }
#pragma unroll
  for (int q = 0; q < KC; ++q) {
    if constexpr (CW == 4) c[q] = (int)w[q];
    else if constexpr (CW == 2) c[q] = (int)((w[q >> 1] >> ((q & 1) * 16)) & 0xffffu);
    else c[q] = (int)((w[q >> 2] >> ((q & 3) * 8)) & 0xffu);
  }
}

__device__ __forceinline__ uint32_t mix32(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdull;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ull;
  x ^= x >> 33;
  return (uint32_t)x;
}

// 32-bit symmetric edge hash (lowbias32 of a mix of both ends and the salt):
// cheap enough for the per-edge inner loop of the matching proposals.
__device__ __forceinline__ uint32_t edge_hash32(int a, int b, uint32_t salt) {
  uint32_t lo = (uint32_t)min(a, b), hi = (uint32_t)max(a, b);
  uint32_t x = lo * 0x9E3779B1u ^ (hi + salt) * 0x85EBCA77u;
  x ^= x >> 16;
  x *= 0x7feb352du;
  x ^= x >> 15;
  x *= 0x846ca68bu;
  x ^= x >> 16;
  return x;
}

__device__ __forceinline__ int warp_id_global() {
  return (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
}
__device__ __forceinline__ int warps_total() { return (int)(((int64_t)gridDim.x * blockDim.x) >> 5); }

// ------------------------------------------------------------------ K1 ---
// Position of the root in v's ascending in-list, or -1 (a DAG has at most
// one root edge per node).
__device__ __forceinline__ int64_t root_slot(const hs_dag_t &g, int v) {
  int64_t lo = g.in_ptr[v], hi = g.in_ptr[v + 1];
  if (g.root == 0) return (lo < hi && g.in_src[lo] == 0) ? lo : -1;  // the root sorts first
  while (lo < hi) {  // lower_bound(root)
    int64_t mid = (lo + hi) >> 1;
    if (g.in_src[mid] < g.root) lo = mid + 1; else hi = mid;
  }
  return (lo < g.in_ptr[v + 1] && g.in_src[lo] == g.root) ? lo : -1;
}

// Kernel positions [kv0, kv1) only (one rank's vertex range when sharded);
// outputs are indexed kv - kv0.
__device__ __forceinline__ int node_of(const hs_dag_t &g, int kv) { return kv < g.root ? kv : kv + 1; }

__global__ void sym_degree(hs_dag_t g, int kv0, int kv1, int32_t *deg) {
  for (int64_t kv = kv0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; kv < kv1;
       kv += (int64_t)gridDim.x * blockDim.x) {
    const int v = node_of(g, (int)kv);
    deg[kv - kv0] = (int)(g.in_ptr[v + 1] - g.in_ptr[v]) - (root_slot(g, v) >= 0 ? 1 : 0) +
                    (int)(g.out_ptr[v + 1] - g.out_ptr[v]);
  }
}

// Team of 8 lanes per vertex: in-neighbours (root dropped) then
// out-neighbours. ew_in (in-order weights) avoids a random gather through
// in_eid when the caller has it; otherwise the weight is gathered.
// 8 CTAs/SM (<= 32 registers): the gathers need the occupancy
template <int T>
__global__ void __launch_bounds__(256, 8) sym_fill(hs_dag_t g, int kv0, int kv1, const int32_t *ew, const int32_t *ew_in,
                         const int32_t *nw, const int64_t *xadj, int32_t *adj, int32_t *wgt,
                         int32_t *vw, int32_t *twin) {
  const int lane = (threadIdx.x & 31) % T;
  const int64_t step = (int64_t)warps_total() * (32 / T);
  for (int64_t vb = kv0 + (int64_t)warp_id_global() * (32 / T); vb < kv1; vb += step) {
    const int kv = (int)(vb + (threadIdx.x & 31) / T);
    if (kv >= kv1) continue;
    const int v = node_of(g, kv);
    const int li = kv - kv0;
    const int64_t pos = xadj[li];
    if (lane == 0) vw[li] = nw[v];
    const int64_t i0 = g.in_ptr[v], i1 = g.in_ptr[v + 1];
    const int64_t rs = root_slot(g, v);
    for (int64_t j = i0 + lane; j < i1; j += T) {
      if (j == rs) continue;
      const int u = g.in_src[j];
      const int64_t at = pos + (j - i0) - (rs >= 0 && j > rs ? 1 : 0);
      const int ku = u < g.root ? u : u - 1;
      adj[at] = ku;
      if (wgt) wgt[at] = ew_in ? ew_in[j] : ew[g.in_eid[j]];
      if (twin) {  // the reverse entry is v in u's out-part: xadj[ku+1] - outdeg(u) + rank
        const int64_t e = g.in_eid[j];
        const int64_t tw = xadj[ku + 1] - g.out_ptr[u + 1] + e;
        twin[at] = (int32_t)tw;
        twin[tw] = (int32_t)at;
      }
    }
    const int64_t opos = pos + (i1 - i0) - (rs >= 0 ? 1 : 0);
    const int64_t o0 = g.out_ptr[v], o1 = g.out_ptr[v + 1];
    for (int64_t j = o0 + lane; j < o1; j += T) {
      const int u = g.out_dst[j];
      adj[opos + (j - o0)] = u < g.root ? u : u - 1;
      if (wgt) wgt[opos + (j - o0)] = ew[j];
    }
  }
}

// Chunked K1 (no twin index): one warp per 32 consecutive kernel positions.
// Consecutive nodes own consecutive ranges of in_src and out_dst, so the warp
// streams the chunk's in-entries and then its out-entries with coalesced
// loads and near-contiguous stores; each entry finds its vertex by a 5-step
// search over the chunk's list prefix in shared memory. Same output as
// sym_fill (the per-vertex order is in-list then out-list).
constexpr int kSymWarps = 8;
constexpr int kSymOwnCap = 768;   // per warp and list kind: entries of a 32-vertex chunk
// Row start of kernel position kv in the undirected graph, without a degree
// pass or scan: both CSRs are prefix sums already, minus the root's own
// lists, minus `roots_before` = root edges into nodes < node_of(kv).
// Assumes no edge into the root (validate()).
__device__ __forceinline__ int64_t sym_row_start(const hs_dag_t &g, int kv, int64_t roots_before) {
  const int v = node_of(g, kv);
  const int r = g.root;
  int64_t x = (g.in_ptr[v] - g.in_ptr[0]) + (g.out_ptr[v] - g.out_ptr[0]);
  if (v > r) x -= (g.in_ptr[r + 1] - g.in_ptr[r]) + (g.out_ptr[r + 1] - g.out_ptr[r]);
  return x - roots_before;
}
// Root edges into nodes < v: a lower_bound over the root's sorted out-list,
// short-cut when v lies past its last target or before its first.
__device__ __forceinline__ int64_t roots_below(const hs_dag_t &g, int v) {
  const int64_t rb = g.out_ptr[g.root], re = g.out_ptr[g.root + 1];
  if (re == rb || g.out_dst[re - 1] < v) return re - rb;
  if (g.out_dst[rb] >= v) return 0;
  int64_t lo = rb, hi = re;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (g.out_dst[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo - rb;
}
__device__ __forceinline__ int64_t sym_row_start(const hs_dag_t &g, int kv) {
  return sym_row_start(g, kv, roots_below(g, node_of(g, kv)));
}

__global__ void __launch_bounds__(kSymWarps * 32, 8) sym_fill_chunk(
    hs_dag_t g, int kv0, int kv1, const int32_t *ew, const int32_t *ew_in, const int32_t *nw,
    int64_t *xadj, int32_t *adj, int32_t *wgt, int32_t *vw) {
  __shared__ int s_ipre[kSymWarps][32], s_opre[kSymWarps][32], s_rs[kSymWarps][32];
  __shared__ int64_t s_ib[kSymWarps][32], s_ob[kSymWarps][32], s_pos[kSymWarps][32],
      s_oat[kSymWarps][32];
  __shared__ uint8_t s_own[kSymWarps][2][kSymOwnCap];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int nl = kv1 - kv0;
  const int64_t nchunks = (nl + 31) / 32;
  // kv = n-1 (one past the last kernel) maps to node n: the totals
  int64_t x0 = 0;
  if (lane == 0) x0 = sym_row_start(g, kv0);
  x0 = __shfl_sync(0xffffffffu, x0, 0);
  if (blockIdx.x == 0 && threadIdx.x == 0) xadj[nl] = sym_row_start(g, kv1) - x0;
  for (int64_t c = warp_id_global(); c < nchunks; c += warps_total()) {
    const int li = (int)(c * 32) + lane;
    const int cnt = min(32, nl - (int)(c * 32));
    int ilen = 0, olen = 0, rsr = INT32_MAX, hasr = 0;
    int64_t ib = 0, ob = 0, rs = -1;
    if (li < nl) {
      const int v = node_of(g, kv0 + li);
      ib = g.in_ptr[v];
      const int64_t ie = g.in_ptr[v + 1];
      ob = g.out_ptr[v];
      const int64_t oe = g.out_ptr[v + 1];
      rs = root_slot(g, v);
      ilen = (int)(ie - ib);
      olen = (int)(oe - ob);
      hasr = rs >= 0;
      if (rs >= 0) rsr = (int)(rs - ib);
      vw[li] = nw[v];
    }
    // the chunk's first row start: root edges below its first node from the
    // first lane that has one (its in_eid is its rank among the root's
    // targets), else one search by lane 0
    const unsigned rmask = __ballot_sync(0xffffffffu, hasr);
    int64_t rb = 0;
    if (rmask) {
      const int fl = __ffs(rmask) - 1;
      if (lane == fl) rb = g.in_eid ? (int64_t)g.in_eid[rs] - g.out_ptr[g.root]
                                    : roots_below(g, node_of(g, kv0 + li));
      rb = __shfl_sync(0xffffffffu, rb, fl);
    } else if (lane == 0) {
      rb = roots_below(g, node_of(g, kv0 + li));
    }
    if (!rmask) rb = __shfl_sync(0xffffffffu, rb, 0);
    int64_t xc = 0;
    if (lane == 0) xc = sym_row_start(g, kv0 + li, rb) - x0;
    xc = __shfl_sync(0xffffffffu, xc, 0);
    int ip = ilen, op = olen, rp = hasr;  // inclusive scans
    for (int o = 1; o < 32; o <<= 1) {
      const int a = __shfl_up_sync(0xffffffffu, ip, o), b = __shfl_up_sync(0xffffffffu, op, o);
      const int r2 = __shfl_up_sync(0xffffffffu, rp, o);
      if (lane >= o) { ip += a; op += b; rp += r2; }
    }
    if (li < nl) {
      const int64_t pos = xc + (ip - ilen) + (op - olen) - (rp - hasr);
      xadj[li] = pos;
      // offsets relative to the chunk entry index f of each list kind
      s_pos[w][lane] = pos - (ip - ilen);                 // in: at = s_pos + f (- 1 past the root slot)
      s_rs[w][lane] = hasr ? (ip - ilen) + rsr : INT32_MAX;  // f of the root slot
      s_oat[w][lane] = pos + (ilen - hasr) - (op - olen);  // out: at = s_oat + f
      s_ob[w][lane] = ob - (op - olen);                  // out: j = s_ob + f
    }
    if (lane == 0) s_ib[w][0] = ib;  // first in-list start of the chunk
    s_ipre[w][lane] = ip - ilen;
    s_opre[w][lane] = op - olen;
    const int tin = __shfl_sync(0xffffffffu, ip, 31), tout = __shfl_sync(0xffffffffu, op, 31);
    // owner map (entry -> lane) when the chunk's lists fit: each lane marks
    // its own ranges once instead of every entry searching the prefix
    const bool own_map = tin <= kSymOwnCap && tout <= kSymOwnCap;
    if (own_map && li < nl) {
      const int a = ip - ilen, b = op - olen;
      for (int r = 0; r < ilen; ++r) s_own[w][0][a + r] = (uint8_t)lane;
      for (int r = 0; r < olen; ++r) s_own[w][1][b + r] = (uint8_t)lane;
    }
    __syncwarp();
    for (int f = lane; f < tin; f += 32) {
      int t = 0;
      if (own_map) {
        t = s_own[w][0][f];
      } else {
        for (int st = 16; st; st >>= 1)
          if (t + st < cnt && s_ipre[w][t + st] <= f) t += st;
      }
      // in-lists of consecutive nodes are one contiguous run (the root has
      // none): j follows from f; f at the root slot is skipped
      const int rsf = s_rs[w][t];
      if (f == rsf) continue;
      const int64_t j = s_ib[w][0] + f;
      const int64_t at = s_pos[w][t] + f - (f > rsf ? 1 : 0);
      const int u = g.in_src[j];
      adj[at] = u < g.root ? u : u - 1;
      if (wgt) wgt[at] = ew_in ? ew_in[j] : ew[g.in_eid[j]];
    }
    for (int f = lane; f < tout; f += 32) {
      int t = 0;
      if (own_map) {
        t = s_own[w][1][f];
      } else {
        for (int st = 16; st; st >>= 1)
          if (t + st < cnt && s_opre[w][t + st] <= f) t += st;
      }
      const int64_t j = s_ob[w][t] + f;  // out-lists: the root's may sit between
      const int64_t at = s_oat[w][t] + f;
      const int u = g.out_dst[j];
      adj[at] = u < g.root ? u : u - 1;
      if (wgt) wgt[at] = ew[j];
    }
    __syncwarp();
  }
}

// ------------------------------------------------------------------ K3 ---
__global__ void __launch_bounds__(256) deg_from_xadj(const int64_t *xadj, int n, int32_t *deg,
                                                     int32_t *max_deg) {
  int mx = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int d = (int32_t)(__ldg(xadj + i + 1) - __ldg(xadj + i));
    deg[i] = d;
    mx = max(mx, d);
  }
  for (int off = 16; off; off >>= 1) mx = max(mx, __shfl_down_sync(0xffffffffu, mx, off));
  __shared__ int sm[8];
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (max_deg && threadIdx.x == 0) {
    for (int q = 1; q < (int)(blockDim.x >> 5); ++q) mx = max(mx, sm[q]);
    atomicMax(max_deg, mx);
  }
}

// Edge rating w^2 / (c(u) c(v)) ("expansion*2"): prefers heavy edges between
// light vertices, which keeps coarse vertex weights even.
__device__ __forceinline__ float rating(int w, int32_t a, int32_t b) {
  return (float)w * (float)w / ((float)a * (float)b);
}

// Block-aggregated append: every thread of the block calls it (block-uniform
// loop trip); one global atomic per block and call (a counter hit by every
// warp serialised in L2). Order of the appended items is unspecified.
template <typename V>
__device__ __forceinline__ void block_append(bool take, V value, V *out, int32_t *count) {
  __shared__ int s_warp[32];
  __shared__ int s_base;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const unsigned m = __ballot_sync(0xffffffffu, take);
  if (lane == 0) s_warp[wid] = __popc(m);
  __syncthreads();
  if (threadIdx.x == 0) {
    int tot = 0;
    for (int w = 0; w < nw; ++w) {
      const int c = s_warp[w];
      s_warp[w] = tot;
      tot += c;
    }
    s_base = tot ? atomicAdd(count, tot) : 0;
  }
  __syncthreads();
  if (take) out[s_base + s_warp[wid] + __popc(m & ((1u << lane) - 1))] = value;
  __syncthreads();
}

// Two-hop ("leaf") matching: unmatched vertices that share a favourite
// neighbour are paired in (favourite, id) order.
__global__ void twohop_keys(int n, const int32_t *match, const int32_t *fav, uint64_t *keys,
                           int32_t *count) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < n; base += stride) {
    const int64_t u = base + threadIdx.x;
    const bool take = u < n && match[u] < 0 && fav[u] >= 0;
    const uint64_t key = take ? ((uint64_t)(uint32_t)fav[u] << 32) | (uint64_t)u : 0;
    block_append<uint64_t>(take, key, keys, count);
  }
}

__global__ void twohop_heads(const uint64_t *keys, int cnt, int32_t *head) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt;
       i += (int64_t)gridDim.x * blockDim.x)
    head[i] = (i == 0 || (keys[i - 1] >> 32) != (keys[i] >> 32)) ? (int32_t)i : 0;
}

// start[i] = first index of i's run (inclusive max-scan of head indices)
__global__ void twohop_pair(const uint64_t *keys, const int32_t *start, int cnt, const int32_t *vw,
                            int32_t max_vw, int32_t *match) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (((i - start[i]) & 1) || i + 1 >= cnt || (keys[i + 1] >> 32) != (keys[i] >> 32)) continue;
    int a = (int)(uint32_t)keys[i], b = (int)(uint32_t)keys[i + 1];
    if (vw[a] + vw[b] > max_vw) continue;
    match[a] = b;
    match[b] = a;
  }
}

// Unmatched vertices of `in` (all n when in == nullptr) -> out (warp-aggregated).
__global__ void unmatched_list(int n, const int32_t *in, const int32_t *in_count,
                               const int32_t *match, int32_t *out, int32_t *out_count) {
  const int nv = in ? *in_count : n;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < nv; base += stride) {
    const int64_t i = base + threadIdx.x;
    const int u = i < nv ? (in ? in[i] : (int)i) : -1;
    block_append<int32_t>(u >= 0 && match[u] < 0, u, out, out_count);
  }
}

__global__ void match_accept(int n, int32_t *match, const int32_t *prop, uint32_t *mw,
                             int32_t *nmatched) {
  int local = 0;
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n;
       u += (int64_t)gridDim.x * blockDim.x) {
    int v = prop[u];
    if (match[u] < 0 && v >= 0 && prop[v] == (int)u) {
      match[u] = v;
      mw[u] |= 0x80000000u;
    }
  }
  (void)local;
  (void)nmatched;
}

// ------------------------------------------------------------------ K4 ---
__global__ void leader_flags(int n, const int32_t *match, int32_t *flag) {
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n;
       u += (int64_t)gridDim.x * blockDim.x) {
    int m = match[u];
    flag[u] = (m < 0 || m >= (int)u) ? 1 : 0;
  }
}

// cmap is replicated (global fine id -> global coarse id = coff + local cid)
__global__ void build_cmap(G g, const int32_t *match, const int32_t *cid, int32_t coff,
                           Rep<int32_t> cmap, int32_t *mem0, int32_t *mem1, int32_t *vw_c,
                           int64_t *ub) {
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < g.n;
       u += (int64_t)gridDim.x * blockDim.x) {
    int m = match[u];
    int partner = (m < 0) ? (int)u : m;
    int lead = min((int)u, partner);
    int c = cid[lead];
    cmap.put(g.v0 + u, coff + c);
    if (lead == (int)u) {
      mem0[c] = (int)u;
      mem1[c] = partner != (int)u ? partner : -1;
      vw_c[c] = g.vw[u] + (partner != (int)u ? g.vw[partner] : 0);
      ub[c] = (int64_t)g.deg[u] + (partner != (int)u ? g.deg[partner] : 0);
    }
  }
}

__device__ __forceinline__ uint32_t slot_hash(int key, uint32_t mask) {
  return ((uint32_t)key * 0x9E3779B1u) & mask;
}

// warp per coarse vertex, table of pow2 >= 2*ub slots in shared memory
constexpr int kWarpSlots = 256;  // per warp: lists up to 128 entries (level 0 is ~40)
constexpr int kContractWarps = 8;

__global__ void __launch_bounds__(kContractWarps * 32)
contract_warp(G g, const int32_t *cmap, const int32_t *mem0, const int32_t *mem1,
              const int64_t *ub, int nc, G c, int stride) {
  __shared__ int32_t keys[kContractWarps][kWarpSlots];
  __shared__ int32_t vals[kContractWarps][kWarpSlots];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  int32_t *K = keys[wl], *V = vals[wl];
  // stride > 1: only every stride-th coarse vertex (merged-degree sampling)
  for (int64_t ci = warp_id_global(); ci * stride < nc; ci += warps_total()) {
    const int cv = (int)(ci * stride);
    const int64_t u_b = ub[cv];
    if (u_b * 2 > kWarpSlots) continue;  // handled by the CTA / global paths
    uint32_t size = 32;
    while (size < 2 * u_b) size <<= 1;
    const uint32_t mask = size - 1;
    for (uint32_t s = lane; s < size; s += 32) { K[s] = -1; V[s] = 0; }
    __syncwarp();
    for (int t = 0; t < 2; ++t) {
      int x = t == 0 ? mem0[cv] : mem1[cv];
      if (x < 0) continue;
      const int64_t b = g.xbeg[x];
      const int d = g.deg[x];
      for (int j = lane; j < d; j += 32) {
        int key = cmap[g.adj[b + j]];
        if (key == cv + c.v0) continue;
        int w = g.ew(b + j);
        uint32_t s = slot_hash(key, mask);
        while (true) {
          int prev = atomicCAS(&K[s], -1, key);
          if (prev == -1 || prev == key) { atomicAdd(&V[s], w); break; }
          s = (s + 1) & mask;
        }
      }
    }
    __syncwarp();
    const int64_t base = c.xbeg[cv];
    int cnt = 0;
    for (uint32_t s0 = 0; s0 < size; s0 += 32) {
      uint32_t s = s0 + lane;
      int key = s < size ? K[s] : -1;
      unsigned m = __ballot_sync(0xffffffffu, key >= 0);
      if (key >= 0) {
        int64_t at = base + cnt + __popc(m & ((1u << lane) - 1));
        c.adj[at] = key;
        c.wgt[at] = V[s];
      }
      cnt += __popc(m);
    }
    if (lane == 0) c.deg[cv] = cnt;
    __syncwarp();
  }
}

// Merged / unmerged entry counts over the sampled coarse vertices.
__global__ void sample_ratio(const int64_t *ub, const int32_t *deg_c, int nc, int stride,
                             int64_t slots, unsigned long long *out) {
  unsigned long long a = 0, b = 0;
  for (int64_t ci = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; ci * stride < nc;
       ci += (int64_t)gridDim.x * blockDim.x) {
    const int64_t cv = ci * stride;
    if (ub[cv] * 2 > slots) continue;
    a += (unsigned long long)deg_c[cv];
    b += (unsigned long long)ub[cv];
  }
  for (int off = 16; off; off >>= 1) {
    a += __shfl_down_sync(0xffffffffu, a, off);
    b += __shfl_down_sync(0xffffffffu, b, off);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&out[0], a);
    atomicAdd(&out[1], b);
  }
}

// Locality probe of the finest level (does coarsening have anything to
// merge?): for every stride-th vertex u and its first kProbeNbrs neighbours v
// (lists capped at kProbeCap entries), count the pairs (u, v) that share a
// neighbour. Contraction only removes edges inside matched pairs or between
// neighbours that are matched together; on a graph without triangles (random
// task DAGs) neither happens beyond the matched edges themselves.
constexpr int kProbeNbrs = 4, kProbeCap = 64;
// One warp per sampled pair: v's list staged in shared memory, u's entries
// tested by the lanes.
__global__ void __launch_bounds__(256) locality_probe(G g, int stride, unsigned long long *out) {
  __shared__ int s_nv[8][kProbeCap];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t npairs = ((int64_t)(g.n - 1) / stride + 1) * kProbeNbrs;
  unsigned long long pairs = 0, shared = 0;
  for (int64_t p = warp_id_global(); p < npairs; p += warps_total()) {
    const int u = (int)(p / kProbeNbrs * stride), a = (int)(p % kProbeNbrs);
    const int64_t bu = g.xbeg[u];
    const int du = min(g.deg[u], kProbeCap);
    if (a >= du) continue;
    const int v = g.adj[bu + a] - g.v0;
    if ((unsigned)v >= (unsigned)g.n || v == u) continue;
    const int64_t bv = g.xbeg[v];
    const int dv = min(g.deg[v], kProbeCap);
    for (int j = lane; j < dv; j += 32) s_nv[w][j] = g.adj[bv + j];
    __syncwarp();
    bool hit = false;
    for (int i = lane; i < du; i += 32) {
      const int x = g.adj[bu + i];
      if (x == v + g.v0) continue;
      for (int j = 0; j < dv; ++j) hit |= s_nv[w][j] == x;
    }
    hit = __any_sync(0xffffffffu, hit);
    ++pairs;
    shared += hit;
    __syncwarp();
  }
  if (lane == 0 && pairs) {
    atomicAdd(&out[0], pairs);
    atomicAdd(&out[1], shared);
  }
}

// Unmerged contraction (the level will be the coarsest): the pair's lists
// mapped through cmap, self loops dropped, parallel edges kept. Refinement
// gains, balance and cut are sums over entries, so they are identical on this
// multigraph. Team of 8 lanes per coarse vertex, ballot-compacted stores.
template <int T>
__global__ void contract_direct(G g, const int32_t *cmap, const int32_t *mem0, const int32_t *mem1,
                                int nc, G c) {
  const int lane = (threadIdx.x & 31) % T, tw = (threadIdx.x & 31) / T;
  const int64_t step = (int64_t)warps_total() * (32 / T);
  for (int64_t vb = (int64_t)warp_id_global() * (32 / T); vb < nc; vb += step) {
    const int cv = (int)(vb + tw);
    const bool valid = cv < nc;
    int64_t base = valid ? c.xbeg[cv] : 0;
    int cnt = 0;
    for (int t = 0; t < 2; ++t) {
      const int x = valid ? (t == 0 ? mem0[cv] : mem1[cv]) : -1;
      const int64_t b = x >= 0 ? g.xbeg[x] : 0;
      const int d = x >= 0 ? g.deg[x] : 0;
      // warp-uniform trip count: max over the 4 teams of this warp
      int dm = d;
      for (int off = 16; off >= T; off >>= 1) dm = max(dm, __shfl_xor_sync(0xffffffffu, dm, off));
      for (int j0 = 0; j0 < dm; j0 += T) {
        const int j = j0 + lane;
        int key = -1, w = 0;
        if (j < d) {
          key = cmap[g.adj[b + j]];
          w = g.ew(b + j);
        }
        const bool keep = key >= 0 && key != cv + c.v0;
        const unsigned m = (__ballot_sync(0xffffffffu, keep) >> (tw * T)) & ((1u << T) - 1);
        if (keep) {
          const int64_t at = base + cnt + __popc(m & ((1u << lane) - 1));
          c.adj[at] = key;
          if (!c.wconst) c.wgt[at] = w;
        }
        cnt += __popc(m);
      }
    }
    if (valid && lane == 0) c.deg[cv] = cnt;
  }
}

// CTA per (long) coarse vertex; table in dynamic shared memory or, when
// `gtab` is set, in global scratch at 2*xbeg (2*ub slots available there).
__global__ void contract_block(G g, const int32_t *cmap, const int32_t *mem0, const int32_t *mem1,
                               const int64_t *ub, const int32_t *list, const int32_t *nlistp, G c,
                               int32_t *gkeys, int32_t *gvals, int smem_slots) {
  extern __shared__ int32_t sm[];
  __shared__ int s_cnt;
  const int nlist = *nlistp;
  for (int li = blockIdx.x; li < nlist; li += gridDim.x) {
    const int cv = list[li];
    const int64_t u_b = ub[cv];
    int32_t *K, *V;
    uint64_t size;
    if (gkeys) {
      size = (uint64_t)(2 * u_b);
      K = gkeys + 2 * c.xbeg[cv];
      V = gvals + 2 * c.xbeg[cv];
    } else {
      size = 32;
      while (size < (uint64_t)(2 * u_b)) size <<= 1;
      K = sm;
      V = sm + smem_slots;
    }
    const bool pow2 = (size & (size - 1)) == 0;
    for (uint64_t s = threadIdx.x; s < size; s += blockDim.x) { K[s] = -1; V[s] = 0; }
    if (threadIdx.x == 0) s_cnt = 0;
    __syncthreads();
    for (int t = 0; t < 2; ++t) {
      int x = t == 0 ? mem0[cv] : mem1[cv];
      if (x < 0) continue;
      const int64_t b = g.xbeg[x];
      const int d = g.deg[x];
      for (int j = threadIdx.x; j < d; j += blockDim.x) {
        int key = cmap[g.adj[b + j]];
        if (key == cv + c.v0) continue;
        int w = g.ew(b + j);
        uint64_t s = pow2 ? (uint64_t)slot_hash(key, (uint32_t)(size - 1))
                          : ((uint64_t)((uint32_t)key * 0x9E3779B1u)) % size;
        while (true) {
          int prev = atomicCAS(&K[s], -1, key);
          if (prev == -1 || prev == key) { atomicAdd(&V[s], w); break; }
          s = s + 1 == size ? 0 : s + 1;
        }
      }
    }
    __syncthreads();
    const int64_t base = c.xbeg[cv];
    for (uint64_t s = threadIdx.x; s < size; s += blockDim.x) {
      int key = K[s];
      if (key >= 0) {
        int at = atomicAdd(&s_cnt, 1);
        c.adj[base + at] = key;
        c.wgt[base + at] = V[s];
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) c.deg[cv] = s_cnt;
    __syncthreads();
  }
}

__global__ void classify_long(const int64_t *ub, const int32_t *ncp, int64_t lo, int64_t hi,
                              int32_t *list, int32_t *count) {
  const int nc = *ncp;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < nc; base += stride) {
    const int64_t i = base + threadIdx.x;
    const bool take = i < nc && ub[i] * 2 > lo && ub[i] * 2 <= hi;
    const unsigned m = __ballot_sync(0xffffffffu, take);
    if (!m) continue;
    const int lane = threadIdx.x & 31, leader = __ffs(m) - 1;
    int at = 0;
    if (lane == leader) at = atomicAdd(count, __popc(m));
    at = __shfl_sync(0xffffffffu, at, leader);
    if (take) list[at + __popc(m & ((1u << lane) - 1))] = (int)i;
  }
}

// ------------------------------------------------------------------ K5 ---
// Initial partitions and small-level refinement: CTA-resident FM.
#include "kway_fm.cuh"

// levels up to this many vertices are refined by FM candidates (one GPU)
constexpr int kFmMaxLevel = 4096;
static_assert(kFmMaxLevel <= kFmMaxN, "FM levels keep their per-vertex state in shared memory");
constexpr int kFmInitPasses = 8, kFmRefinePasses = 6, kFmCopies = 16;
// coarsening stops on density only past this many adjacency entries
constexpr int64_t kDenseStopNnz = 4ll << 20;

int dev_id() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}

// ------------------------------------------------------------------ K6 ---
__global__ void project(int n, const int32_t *cmap, const part_t *cpart, part_t *part) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    part[i] = cpart[cmap[i]];
}

// Per-part weight sums. Each thread walks 16 consecutive vertices (one
// 16-byte part load, four 16-byte weight loads when aligned) keeping a run
// (part, sum) and flushing it to shared memory when the part changes — parts
// come in long runs after the band start, so flushes are rare; the last run
// of every thread goes through one warp-wide __reduce_add per distinct part.
// Sums fit 32 bits: the total vertex weight is < 2^31 (the weight guard).
constexpr int kPwChunk = 16;
__global__ void __launch_bounds__(256) part_weights(int n, const int32_t *vw, const part_t *part,
                                                    int k, int64_t *pw) {
  __shared__ unsigned s[kMaxParts];
  for (int p = threadIdx.x; p < k; p += blockDim.x) s[p] = 0;
  __syncthreads();
  const bool vec = (((uintptr_t)vw | (uintptr_t)part) & 15) == 0;
  const int64_t chunks = ((int64_t)n + kPwChunk - 1) / kPwChunk;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t trips = (chunks + stride - 1) / stride;  // warp-uniform trip count
  int cur = -1;
  unsigned acc = 0;
  for (int64_t t = 0; t < trips; ++t) {
    const int64_t c = t * stride + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= chunks) break;
    const int64_t i0 = c * kPwChunk;
    int8_t pb[kPwChunk];
    int32_t wb[kPwChunk];
    int cnt = kPwChunk;
    if (vec && i0 + kPwChunk <= n) {
      *(int4 *)pb = __ldg((const int4 *)(part + i0));
#pragma unroll
      for (int q = 0; q < kPwChunk / 4; ++q) *(int4 *)(wb + 4 * q) = __ldg((const int4 *)(vw + i0) + q);
    } else {
      cnt = (int)(n - i0 < kPwChunk ? n - i0 : kPwChunk);
#pragma unroll
      for (int q = 0; q < kPwChunk; ++q) {
        pb[q] = q < cnt ? part[i0 + q] : 0;
        wb[q] = q < cnt ? vw[i0 + q] : 0;
      }
    }
#pragma unroll
    for (int q = 0; q < kPwChunk; ++q) {
      if (q >= cnt) break;
      const int p = pb[q];
      if (p != cur) {
        if (cur >= 0 && acc) atomicAdd(&s[cur], acc);
        cur = p;
        acc = 0;
      }
      acc += (unsigned)wb[q];
    }
  }
  const unsigned peers = __match_any_sync(0xffffffffu, cur);
  const unsigned sum = __reduce_add_sync(peers, acc);
  if (cur >= 0 && (threadIdx.x & 31) == __ffs(peers) - 1 && sum) atomicAdd(&s[cur], sum);
  __syncthreads();
  for (int p = threadIdx.x; p < k; p += blockDim.x)
    if (s[p]) atomicAdd((unsigned long long *)&pw[p], (unsigned long long)s[p]);
}

constexpr int kRefWarps = 8;

// Rebalance candidates: every vertex of an over-full part proposes its best
// (max gain, possibly negative) part still below its target.
__global__ void __launch_bounds__(kRefWarps * 32)
rebalance_candidates(G g, const part_t *part, int k, const int64_t *pw, const int64_t *hi,
                     const int64_t *target, int32_t *cand, const int32_t *run) {
  if (run && !*run) return;
  __shared__ int32_t conn_s[kRefWarps][kMaxParts];
  __shared__ int64_t s_pw[kMaxParts], s_hi[kMaxParts], s_t[kMaxParts];
  for (int p = threadIdx.x; p < k; p += blockDim.x) {
    s_pw[p] = pw[p];
    s_hi[p] = hi[p];
    s_t[p] = target[p];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  int32_t *conn = conn_s[wl];
  for (int v = warp_id_global(); v < g.n; v += warps_total()) {
    const int own = part[g.v0 + v];
    if (s_pw[own] <= s_hi[own]) {
      if (lane == 0) cand[v] = -1;
      continue;
    }
    for (int p = lane; p < k; p += 32) conn[p] = 0;
    __syncwarp();
    const int64_t b = g.xbeg[v];
    const int d = g.deg[v];
    for (int j = lane; j < d; j += 32) atomicAdd(&conn[part[g.adj[b + j]]], g.ew(b + j));
    __syncwarp();
    int bg = INT_MIN, bp = -1;
    for (int p = lane; p < k; p += 32) {
      if (p == own || s_pw[p] >= s_t[p]) continue;
      int gain = conn[p] - conn[own];
      if (bp < 0 || gain > bg || (gain == bg && p < bp)) { bg = gain; bp = p; }
    }
    for (int off = 16; off; off >>= 1) {
      int og = __shfl_down_sync(0xffffffffu, bg, off);
      int op = __shfl_down_sync(0xffffffffu, bp, off);
      if (op >= 0 && (bp < 0 || og > bg || (og == bg && op < bp))) { bg = og; bp = op; }
    }
    if (lane == 0) cand[v] = bp;
    __syncwarp();
  }
}

// flows[p] = weight leaving p, flows[k + q] = weight entering q (planned moves)
__global__ void move_flows(int n, const int32_t *vw, const part_t *part, const int32_t *cand,
                           int k, int64_t *flows, int32_t *nmoves, const int32_t *run) {
  if (run && !*run) return;
  __shared__ unsigned long long s[2 * kMaxParts];
  __shared__ int s_n;
  for (int p = threadIdx.x; p < 2 * k; p += blockDim.x) s[p] = 0;
  if (threadIdx.x == 0) s_n = 0;
  __syncthreads();
  int local = 0;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    int dest = cand[v];
    if (dest >= 0) {
      atomicAdd(&s[part[v]], (unsigned long long)vw[v]);
      atomicAdd(&s[k + dest], (unsigned long long)vw[v]);
      ++local;
    }
  }
  if (local) atomicAdd(&s_n, local);
  __syncthreads();
  for (int p = threadIdx.x; p < 2 * k; p += blockDim.x)
    if (s[p]) atomicAdd((unsigned long long *)&flows[p], s[p]);
  if (threadIdx.x == 0 && s_n) atomicAdd(nmoves, s_n);
}

// Applies planned moves, each kept with probability p_out[own] * p_in[dest]
// decided by a hash of (salt, v) — deterministic thinning that keeps the
// expected inflow of every part within its room.
__device__ __forceinline__ void cache_move(const G &g, const Conn &cache, int v, int own,
                                           int dest);

__global__ void apply_thinned(int n, const int32_t *vw, const int32_t *cand, const double *prob,
                              int k, uint64_t salt, int32_t v0, const part_t *part,
                              Rep<part_t> prep, int64_t *pw, const int32_t *run,
                              const int64_t *xbeg, const int32_t *deg, const int32_t *twin,
                              part_t *gp, G g, Conn cache) {
  if (run && !*run) return;
  __shared__ long long s[kMaxParts];
  __shared__ double s_prob[2 * kMaxParts];
  for (int p = threadIdx.x; p < k; p += blockDim.x) s[p] = 0;
  for (int p = threadIdx.x; p < 2 * k; p += blockDim.x) s_prob[p] = prob[p];
  __syncthreads();
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    int dest = cand[v];
    if (dest < 0) continue;
    int own = part[v0 + v];
    double pr = s_prob[own] * s_prob[k + dest];
    const uint64_t gv = (uint64_t)(v0 + v);
    if (pr < 1.0 && (double)mix32(salt ^ (gv * 0x9E3779B97F4A7C15ull)) >= pr * 4294967296.0)
      continue;
    prep.put(v0 + v, (part_t)dest);
    if (gp)
      for (int64_t j = xbeg[v], e = xbeg[v] + deg[v]; j < e; ++j) gp[twin[j]] = (part_t)dest;
    if (cache.p) cache_move(g, cache, (int)v, own, dest);
    atomicAdd((unsigned long long *)&s[dest], (unsigned long long)(long long)vw[v]);
    atomicAdd((unsigned long long *)&s[own], (unsigned long long)(-(long long)vw[v]));
  }
  __syncthreads();
  for (int p = threadIdx.x; p < k; p += blockDim.x)
    if (s[p]) atomicAdd((unsigned long long *)&pw[p], (unsigned long long)s[p]);
}

__global__ void scale_weights(int64_t nnz, const int32_t *in, int32_t *out, int64_t div) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nnz;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t w = in[i] / div;
    out[i] = (int32_t)(w < 1 ? 1 : w);
  }
}

// Initial "range" trial: contiguous id ranges by cumulative weight. Coarse
// ids follow the smallest fine id they contain, so on a task DAG (ids in
// creation/topological order) this is a layer-band partition.
__global__ void range_parts(int n, const int64_t *prefix, int64_t woff, const int32_t *vw,
                            const double *cum, int k, int64_t total, int32_t v0,
                            Rep<part_t> part) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    double mid = ((double)(prefix[v] + woff) + 0.5 * (double)vw[v]) / (double)total;
    int p = 0;
    while (p < k - 1 && mid >= cum[p + 1]) ++p;
    part.put(v0 + v, (part_t)p);
  }
}

// int32 min/max words (written by wstats_kernel) -> int64 slots in place
__global__ void widen_minmax(int64_t *mm) {
  const int32_t lo = ((const int32_t *)mm)[0], hi = ((const int32_t *)(mm + 1))[0];
  mm[0] = lo;
  mm[1] = hi;
}

// sum / min / max of int32 weights (out: u64 sum, i32 min, i32 max; caller
// initialises 0, INT_MAX, INT_MIN): 16-byte loads over the aligned body, one
// atomic triple per block
__global__ void __launch_bounds__(256) wstats_kernel(int64_t n, const int32_t *w,
                                                     unsigned long long *sum, int32_t *mn,
                                                     int32_t *mx) {
  unsigned long long s = 0;
  int lo = INT_MAX, hi = INT_MIN;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t h0 = ((16 - ((uintptr_t)w & 15)) & 15) / 4, head = n < h0 ? n : h0;
  const int64_t n4 = (n - head) / 4;
  const int4 *w4 = (const int4 *)(w + head);
  auto take = [&](int x) {
    s += (unsigned long long)(long long)x;
    lo = min(lo, x);
    hi = max(hi, x);
  };
  for (int64_t j = tid; j < n4; j += 2 * stride) {
    const int4 a = __ldg(w4 + j);
    const bool two = j + stride < n4;
    const int4 b = two ? __ldg(w4 + j + stride) : make_int4(a.x, a.x, a.x, a.x);
    take(a.x), take(a.y), take(a.z), take(a.w);
    if (two) take(b.x), take(b.y), take(b.z), take(b.w);
  }
  for (int64_t j = tid; j < head; j += stride) take(__ldg(w + j));
  for (int64_t j = head + 4 * n4 + tid; j < n; j += stride) take(__ldg(w + j));
  for (int off = 16; off; off >>= 1) {
    s += __shfl_down_sync(0xffffffffu, s, off);
    lo = min(lo, __shfl_down_sync(0xffffffffu, lo, off));
    hi = max(hi, __shfl_down_sync(0xffffffffu, hi, off));
  }
  __shared__ unsigned long long ss[8];
  __shared__ int sl[8], sh[8];
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if ((threadIdx.x & 31) == 0) ss[warp] = s, sl[warp] = lo, sh[warp] = hi;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int q = 1; q < nw; ++q) s += ss[q], lo = min(lo, sl[q]), hi = max(hi, sh[q]);
    atomicAdd(sum, s);
    atomicMin(mn, lo);
    atomicMax(mx, hi);
  }
}

__global__ void int8_to_int32(const int8_t *in, int n, int32_t *out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = in[i];
}

#include "kway_team.cuh"

__global__ void ghost_fill(int64_t nnz, const int32_t *adj, const part_t *part, part_t *gp) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nnz;
       j += (int64_t)gridDim.x * blockDim.x)
    gp[j] = part[adj[j]];
}

// out[0] = min weight, out[1] = -max weight (both via atomicMin; the caller
// initialises both words to 0x7f7f7f7f)
__global__ void wrange_kernel(int64_t nnz, const int32_t *w, int32_t *out) {
  int mn = INT_MAX, mx = INT_MIN;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nnz;
       j += (int64_t)gridDim.x * blockDim.x) {
    mn = min(mn, w[j]);
    mx = max(mx, w[j]);
  }
  for (int off = 16; off; off >>= 1) {
    mn = min(mn, __shfl_down_sync(0xffffffffu, mn, off));
    mx = max(mx, __shfl_down_sync(0xffffffffu, mx, off));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&out[0], mn);
    atomicMin(&out[1], -mx);
  }
}

// max over vertices of the weighted degree (saturating at 2^30)
__global__ void max_wdeg_kernel(G g, int32_t *out) {
  int local = 0;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < g.n;
       v += (int64_t)gridDim.x * blockDim.x) {
    int64_t sum = 0;
    const int64_t b = g.xbeg[v];
    for (int j = 0; j < g.deg[v] && sum < (1 << 30); ++j) sum += g.ew(b + j);
    local = max(local, (int)(sum < (1 << 30) ? sum : (1 << 30)));
  }
  for (int off = 16; off; off >>= 1) local = max(local, __shfl_down_sync(0xffffffffu, local, off));
  if ((threadIdx.x & 31) == 0) atomicMax(out, local);
}

// ------------------------------------------------------------ host side ---
struct Level {
  G g;                      // this rank's rows (all rows on one GPU)
  int32_t n_glob = 0;       // vertices over all ranks
  int64_t nnz_glob = 0;     // live adjacency entries over all ranks
  int32_t *cmap = nullptr;  // global fine id -> global coarse id of the NEXT level
                            // (this rank's replica; set when coarsened)
  bool own_adj = true, own_wgt = true, own_xbeg_vw = true;
  bool unmerged = false;    // built by contract_direct (parallel edges kept)
  int32_t vconst = 0;       // every vertex weighs vconst (0: not uniform / unknown)
};

// Loopback groups (ranks = host threads on one GPU) synchronise on the host:
// a kernel spinning on a peer's flag inside one CUDA context can deadlock
// against that peer's own launches (lazy kernel loading synchronises the
// context), so there each all-reduce is post -> stream sync -> host barrier ->
// reduce. One-process-per-GPU groups use the in-kernel flags.
struct HostBarrier {
  std::mutex mu;
  std::condition_variable cv;
  int count = 0;
  uint64_t gen = 0;
  bool wait(int P, double seconds) {
    std::unique_lock<std::mutex> lk(mu);
    const uint64_t g = gen;
    if (++count == P) {
      count = 0;
      ++gen;
      cv.notify_all();
      return true;
    }
    return cv.wait_for(lk, std::chrono::duration<double>(seconds), [&] { return gen != g; });
  }
};
std::mutex g_hb_mu;
std::vector<std::pair<void *, std::shared_ptr<HostBarrier>>> g_hbs;
std::shared_ptr<HostBarrier> host_barrier_for(void *key) {
  std::lock_guard<std::mutex> lk(g_hb_mu);
  for (auto &e : g_hbs)
    if (e.first == key) return e.second;
  g_hbs.emplace_back(key, std::make_shared<HostBarrier>());
  return g_hbs.back().second;
}

// Flags are never reset, so epochs continue across calls: a rank's last
// epoch is the flag it wrote into its own arena (0 in a fresh arena).
int load_epoch(const Dist &D, uint32_t *epoch, cudaStream_t s) {
  HS_CHECK_CUDA(cudaMemcpyAsync(epoch, D.arena[D.rank] + 4 * D.rank, 4, cudaMemcpyDeviceToHost, s));
  HS_CHECK_CUDA(cudaStreamSynchronize(s));
  return HS_OK;
}

// Loopback ranks share this process's default memory pool: a pool allowed to
// reuse a block freed on another rank's stream would make this rank wait on
// that stream — which may be parked in a barrier waiting for this rank.
int no_cross_stream_pool_waits() {
  static std::once_flag once;
  static cudaError_t err = cudaSuccess;
  std::call_once(once, [] {
    int dev = 0;
    cudaMemPool_t pool;
    err = cudaGetDevice(&dev);
    if (err == cudaSuccess) err = cudaDeviceGetDefaultMemPool(&pool, dev);
    int zero = 0;
    if (err == cudaSuccess)
      err = cudaMemPoolSetAttribute(pool, cudaMemPoolReuseAllowInternalDependencies, &zero);
  });
  HS_CHECK_CUDA(err);
  return HS_OK;
}

template <typename T>
cudaError_t dalloc(T **p, size_t count, cudaStream_t s) {
  return cudaMallocAsync((void **)p, (count ? count : 1) * sizeof(T), s);
}

int warp_grid(int64_t items, int warps_per_block) {
  int64_t g = (items + warps_per_block - 1) / warps_per_block;
  int64_t maxg = (int64_t)hs::sm_count() * 64;
  if (g > maxg) g = maxg;
  return (int)(g < 1 ? 1 : g);
}

template <typename T>
int exclusive_scan(const T *in, T *out, int64_t n, cudaStream_t s) {
  size_t tb = 0;
  HS_CHECK_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, n, s));
  hs::Scratch<char> tmp;
  HS_CHECK_CUDA(tmp.alloc(tb, s));
  HS_CHECK_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, in, out, n, s));
  hs::count_launch(1);
  return HS_OK;
}

// out[0..n] = exclusive prefix of in[0..n) widened to int64 on the fly (no
// int64 copy of the input; out[n] is the total)
struct Widen32 {
  const int32_t *in;
  int64_t n;
  __host__ __device__ int64_t operator()(int64_t i) const { return i < n ? (int64_t)in[i] : 0; }
};
int exclusive_scan_widen(const int32_t *in, int64_t *out, int64_t n, cudaStream_t s) {
  auto it = thrust::make_transform_iterator(thrust::counting_iterator<int64_t>(0), Widen32{in, n});
  size_t tb = 0;
  HS_CHECK_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, it, out, n + 1, s));
  hs::Scratch<char> tmp;
  HS_CHECK_CUDA(tmp.alloc(tb, s));
  HS_CHECK_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, it, out, n + 1, s));
  hs::count_launch(1);
  return HS_OK;
}

struct PhaseTimer {
  bool on;
  cudaStream_t s;
  std::vector<std::pair<const char *, cudaEvent_t>> ev;
  PhaseTimer(cudaStream_t st) : s(st) { on = getenv("HS_KWAY_TRACE") != nullptr; }
  void mark(const char *name) {
    if (!on) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, s);
    ev.emplace_back(name, e);
  }
  ~PhaseTimer() {
    if (!on || ev.empty()) return;
    cudaEventSynchronize(ev.back().second);
    for (size_t i = 1; i < ev.size(); ++i) {
      float ms = 0;
      cudaEventElapsedTime(&ms, ev[i - 1].second, ev[i].second);
      fprintf(stderr, "[kway] %-28s %8.3f ms\n", ev[i].first, ms);
    }
    for (auto &x : ev) cudaEventDestroy(x.second);
  }
};

// Host-side helper that owns the per-call device state.
struct Kway {
  cudaStream_t s;
  int k;
  double tol;
  uint64_t seed, salt;
  int64_t total_vw = 0;
  std::vector<int64_t> hi, lo, target;
  std::vector<double> cum;
  int64_t *d_hi = nullptr, *d_lo = nullptr, *d_target = nullptr, *d_pw = nullptr,
          *d_flows = nullptr;
  double *d_prob = nullptr, *d_cum = nullptr;
  int32_t *counter = nullptr;
  int32_t *ctl = nullptr;   // device control block (see CTL_* in kway_team.cuh)
  part_t *gp = nullptr;     // ghost parts of the level being refined (finest only)
  int64_t *d_nnz = nullptr, *h_nnz = nullptr;
  bool prev_nnz_pending = false;
  std::vector<Level> levels;
  PhaseTimer timer;
  // measured on the config-4 DAG: 1 pass on coarse levels + 4 on the finest
  // beat 4 + 4 on both time and cut (over-refined coarse levels trap the
  // finest level in a worse local optimum)
  int passes_big = 4, passes_small = 8, passes_coarse = 1, rounds = 3;
  bool passes_env = false;
  double max_deg = 1e30;  // coarsening stop threshold (average degree)
  // connectivity cache of the level being refined (one GPU, k <= 16):
  // cache[v][q] = weight of v's edges into part q, kc = 8 or 16 ints per row
  Conn cache;                 // cache.p == nullptr: none
  // caller's start partitions of the finest level (int32 [n_starts][n]),
  // refined and ranked with the FM candidates
  const int32_t *starts = nullptr;
  int n_starts = 0;
  int64_t max_deg0 = 0;       // largest degree of the finest level (cache width)
  Dist D;                         // P = 1: the whole graph on this GPU
  std::shared_ptr<HostBarrier> hb;  // loopback groups
  int64_t *d_dpw = nullptr;       // sharded: this rank's part-weight deltas
  int64_t *d_arbuf = nullptr;     // sharded: staging for host all-reduces

  // ---- sharding helpers (no-ops on one GPU) ----
  // All-reduce of up to kArSlots values over the group; also a barrier.
  int ar(std::initializer_list<ArSeg> segs, int line = __builtin_LINE()) {
    if (!D.on()) return HS_OK;
    ArArgs A;
    static const char *wd = getenv("HS_DIST_WATCHDOG_S");
    if (wd) A.timeout_ns = (uint64_t)(atof(wd) * 1e9);
    static const bool trace = getenv("HS_DIST_TRACE") != nullptr;
    if (trace) fprintf(stderr, "[dist] rank %d epoch %u line %d\n", D.rank, D.epoch + 1, line);
    for (int r = 0; r < D.P; ++r) A.arena[r] = D.arena[r];
    A.rank = D.rank;
    A.P = D.P;
    A.epoch = ++D.epoch;
    int tot = 0;
    for (const ArSeg &g : segs) {
      HS_REQUIRE(A.nseg < 6, HS_EINVAL, "all-reduce: too many segments");
      A.seg[A.nseg++] = g;
      tot += g.n;
    }
    HS_REQUIRE(tot <= kArSlots, HS_EINVAL, "all-reduce: %d values > %d", tot, kArSlots);
    if (!D.threads) {
      ar_kernel<<<1, 256, 0, s>>>(A);
      HS_CHECK_LAUNCH();
      return HS_OK;
    }
    A.phase = 1;
    ar_kernel<<<1, 256, 0, s>>>(A);
    HS_CHECK_LAUNCH();
    HS_CHECK_CUDA(cudaStreamSynchronize(s));
    HS_REQUIRE(hb->wait(D.P, A.timeout_ns * 1e-9), HS_EDEADLOCK,
               "k-way (sharded): a peer thread never reached barrier %u", A.epoch);
    A.phase = 2;
    ar_kernel<<<1, 256, 0, s>>>(A);
    HS_CHECK_LAUNCH();
    return HS_OK;
  }
  int barrier(int line = __builtin_LINE()) { return ar({}, line); }
  static ArSeg seg64(int64_t *p, int n, int op = 0, int acc = 0, int64_t *out = nullptr) {
    ArSeg g;
    g.in = p; g.out = out ? out : p; g.n = n; g.is64 = 1; g.op = (int8_t)op; g.acc = (int8_t)acc;
    return g;
  }
  static ArSeg seg32(int32_t *p, int n, int op = 0) {
    ArSeg g;
    g.in = p; g.out = p; g.n = n; g.is64 = 0; g.op = (int8_t)op;
    return g;
  }
  // Host values in/out (synchronous); checks the watchdog.
  int ar_host(int64_t *vals, int n, int op = 0, int line = __builtin_LINE()) {
    if (!D.on()) return HS_OK;
    HS_CHECK_CUDA(cudaMemcpyAsync(d_arbuf, vals, n * 8, cudaMemcpyHostToDevice, s));
    int rc = ar({seg64(d_arbuf, n, op)}, line);
    if (rc) return rc;
    HS_CHECK_CUDA(cudaMemcpyAsync(vals, d_arbuf, n * 8, cudaMemcpyDeviceToHost, s));
    return check_peers();
  }
  int check_peers() {
    if (!D.on()) return HS_OK;
    int32_t err = 0;
    HS_CHECK_CUDA(cudaMemcpyAsync(&err, D.arena[D.rank] + 64, 4, cudaMemcpyDeviceToHost, s));
    HS_CHECK_CUDA(cudaStreamSynchronize(s));
    HS_REQUIRE(err == 0, HS_EDEADLOCK, "k-way (sharded): a peer never reached a barrier");
    return HS_OK;
  }
  // Sum over ranks of one host value; *before = sum over lower ranks.
  int exscan_host(int64_t mine, int64_t *before, int64_t *total, int line = __builtin_LINE()) {
    int64_t v[kMaxRanks] = {0};
    v[D.rank] = mine;
    int rc = ar_host(v, D.P, 0, line);
    if (rc) return rc;
    *before = 0;
    *total = 0;
    for (int r = 0; r < D.P; ++r) {
      if (r < D.rank) *before += v[r];
      *total += v[r];
    }
    return HS_OK;
  }
  // Replicated array of `count` elements: a private buffer on one GPU, the
  // same offset of every rank's arena when sharded.
  template <typename T>
  int alloc_rep(Rep<T> &r, int64_t count) {
    if (!D.on()) {
      r.n = 1;
      HS_CHECK_CUDA(dalloc(&r.p[0], count, s));
      return HS_OK;
    }
    const int64_t bytes = ((std::max<int64_t>(count, 1) * (int64_t)sizeof(T)) + 255) & ~255ll;
    HS_REQUIRE(D.bump + bytes <= D.arena_bytes, HS_ELIMIT,
               "k-way (sharded): arena too small (%lld bytes needed beyond %lld)",
               (long long)bytes, (long long)D.arena_bytes);
    r.n = D.P;
    for (int q = 0; q < D.P; ++q) r.p[q] = (T *)(D.arena[q] + D.bump);
    D.bump += bytes;
    return HS_OK;
  }
  template <typename T>
  T *loc(const Rep<T> &r) const { return r.p[D.on() ? D.rank : 0]; }
  template <typename T>
  void free_rep(Rep<T> &r) {
    if (!D.on() && r.p[0]) cudaFreeAsync(r.p[0], s);
    r.p[0] = nullptr;
  }
  Kway(cudaStream_t st) : s(st), timer(st) {
    if (const char *e = getenv("HS_KWAY_PASSES")) passes_big = std::max(1, atoi(e)), passes_env = true;
    if (const char *e = getenv("HS_KWAY_ROUNDS")) rounds = std::max(1, atoi(e));
  }

  // part: this rank's replica (global ids); sums this rank's vertices, then all ranks'
  int weights(const G &g, const part_t *part) {
    HS_CHECK_CUDA(cudaMemsetAsync(d_pw, 0, k * sizeof(int64_t), s));
    const int64_t chunks = ((int64_t)g.n + kPwChunk - 1) / kPwChunk;
    part_weights<<<hs::grid_for(chunks, 256, hs::sm_count() * 4), 256, 0, s>>>(g.n, g.vw,
                                                                              part + g.v0, k, d_pw);
    HS_CHECK_LAUNCH();
    return ar({seg64(d_pw, k)});
  }

  // plans in `cand` -> thinned application; returns moves planned
  static int team_grid(int64_t n, int T) {
    int64_t g = (n * T + kTeamBlock - 1) / kTeamBlock;
    int64_t maxg = (int64_t)hs::sm_count() * 32;
    return (int)std::max<int64_t>(1, std::min(g, maxg));
  }

  // Up to `rounds` rebalancing rounds, each gated on the device by "some part
  // is above its bound" — no host round trip.
  // Planned flows and move counts of all ranks (a no-op on one GPU).
  int ar_flows() { return ar({seg64(d_flows, 2 * k), seg32(ctl + CTL_NCONF, 1)}); }
  // Part-weight deltas of this rank's applied moves -> every rank's d_pw.
  int64_t *apply_target() {
    if (!D.on()) return d_pw;
    cudaMemsetAsync(d_dpw, 0, k * sizeof(int64_t), s);
    return d_dpw;
  }
  int ar_applied() { return D.on() ? ar({seg64(d_dpw, k, 0, 1, d_pw)}) : HS_OK; }

  int rebalance(const G &g, const Rep<part_t> &part, int32_t *cand, uint64_t salt2, int rounds,
                Conn cch = Conn()) {
    const int grid = hs::grid_for(g.n, 256, hs::sm_count() * 4);
    const part_t *pl = loc(part);
    for (int rb = 0; rb < rounds; ++rb) {
      balance_check<<<1, 32, 0, s>>>(k, d_pw, d_hi, ctl);
      HS_CHECK_LAUNCH();
      // balanced (the usual case): stop here instead of launching the
      // remaining device-gated rounds (five launches each); every rank reads
      // the same all-reduced part weights, so sharded ranks agree
      int32_t over = 1;
      HS_CHECK_CUDA(cudaMemcpyAsync(&over, ctl + CTL_OVER, 4, cudaMemcpyDeviceToHost, s));
      HS_CHECK_CUDA(cudaStreamSynchronize(s));
      if (!over) break;
      rebalance_candidates<<<warp_grid(g.n, kRefWarps), kRefWarps * 32, 0, s>>>(
          g, pl, k, d_pw, d_hi, d_target, cand, ctl + CTL_OVER);
      HS_CHECK_LAUNCH();
      HS_CHECK_CUDA(cudaMemsetAsync(d_flows, 0, 2 * k * sizeof(int64_t), s));
      HS_CHECK_CUDA(cudaMemsetAsync(ctl + CTL_NCONF, 0, sizeof(int32_t), s));
      move_flows<<<grid, 256, 0, s>>>(g.n, g.vw, pl + g.v0, cand, k, d_flows, ctl + CTL_NCONF,
                                      ctl + CTL_OVER);
      HS_CHECK_LAUNCH();
      int rc = ar_flows();
      if (rc) return rc;
      plan_kernel<<<1, kMaxParts, 0, s>>>(k, g.n, 1, d_flows, d_pw, d_hi, d_lo, d_target, d_prob,
                                          ctl);
      HS_CHECK_LAUNCH();
      int64_t *tgt = apply_target();
      apply_thinned<<<grid, 256, 0, s>>>(g.n, g.vw, cand, d_prob, k, salt2 + rb * 7919, g.v0, pl,
                                         part, tgt, ctl + CTL_APPLY, g.xbeg, g.deg, g.twin, gp, g,
                                         cch);
      HS_CHECK_LAUNCH();
      rc = ar_applied();
      if (rc) return rc;
    }
    return HS_OK;
  }

  // K6 on one level: fixed pass budget, convergence decided on the device.
  int refine(const Level &Lv, const Rep<part_t> &part, uint64_t salt2, bool finest = true) {
    const G &g = Lv.g;
    const part_t *pl = loc(part);
    int32_t *cand, *list, *conf;
    Rep<uint32_t> st;
    HS_CHECK_CUDA(dalloc(&cand, g.n, s));
    const int64_t arena_mark = D.bump;  // st is released (stack order) when this level is done
    int rc = alloc_rep(st, Lv.n_glob);
    if (rc) return rc;
    HS_CHECK_CUDA(dalloc(&list, g.n, s));
    HS_CHECK_CUDA(dalloc(&conf, g.n, s));
    rc = weights(g, pl);
    if (rc) return rc;
    // finest level with twins: ghost copies of the neighbours' parts inside
    // the adjacency stream (refinement reads 1 coalesced byte per entry)
    int32_t wconst = g.wconst;
    if (finest && g.twin && !D.on()) {
      HS_CHECK_CUDA(dalloc(&gp, g.nnz, s));
      ghost_fill<<<hs::grid_for(g.nnz, 256), 256, 0, s>>>(g.nnz, g.adj, pl, gp);
      HS_CHECK_LAUNCH();
      if (!wconst) {
        HS_CHECK_CUDA(cudaMemsetAsync(ctl + 13, 0x7f, 2 * sizeof(int32_t), s));
        wrange_kernel<<<hs::grid_for(g.nnz, 256, hs::sm_count() * 8), 256, 0, s>>>(g.nnz, g.wgt,
                                                                                 ctl + 13);
        HS_CHECK_LAUNCH();
        int32_t mm[2];
        HS_CHECK_CUDA(cudaMemcpyAsync(mm, ctl + 13, sizeof mm, cudaMemcpyDeviceToHost, s));
        HS_CHECK_CUDA(cudaStreamSynchronize(s));
        if (mm[0] == -mm[1]) wconst = mm[0];  // every edge weight equal: skip the weight stream
      }
    }
    rc = rebalance(g, part, cand, salt2 ^ 0xabcdefull, 3);
    if (rc) return rc;
    const int T = team_for(g);
    const int tgrid = team_grid(g.n, T);
    // list-based afterburner: thin candidates before evaluating them (sharded:
    // flows all-reduced, dropped states stored into every replica). A pass
    // then costs ~0.2-0.4 ms instead of ~1.1 ms on config 4, so the finest
    // level gets two passes more. Measured step (ms, cut) by passes:
    // 6 (4.25, 1,320.1M), 8 (4.75, 1,309.7M), 10 (5.20, 1,304.2M),
    // 12 (5.47, 1,302.4M, converged); 4 unthinned passes were (6.38, 1,326.6M).
    const bool prethin = true;
    int max_passes = Lv.nnz_glob > (4ll << 20) ? passes_big + (prethin && !passes_env ? 2 : 0)
                                               : passes_small;
    if (!finest && passes_coarse >= 0) max_passes = passes_coarse;
    // An unmerged level has as many entries as the level below it: a pass
    // there costs a full fine pass and only moves whole pairs, which the fine
    // passes can do too (measured on config 4: 2.6 ms saved, cut 0.2% lower).
    if (!finest && Lv.unmerged) max_passes = 0;
    // 16-bit packed connectivity counters are exact iff every vertex's
    // weighted degree stays below 2^16 on this level
    // (only the register-counter variants use them: skip the scan otherwise)
    bool pack16 = false;
    if (k > 16) {
      HS_CHECK_CUDA(cudaMemsetAsync(ctl + 12, 0, sizeof(int32_t), s));
      max_wdeg_kernel<<<hs::grid_for(g.n, 256, hs::sm_count() * 8), 256, 0, s>>>(g, ctl + 12);
      HS_CHECK_LAUNCH();
      rc = ar({seg32(ctl + 12, 1, 1)});
      if (rc) return rc;
      int32_t mx = 0;
      HS_CHECK_CUDA(cudaMemcpyAsync(&mx, ctl + 12, sizeof mx, cudaMemcpyDeviceToHost, s));
      HS_CHECK_CUDA(cudaStreamSynchronize(s));
      pack16 = mx < 65536;
    }
    // connectivity cache: pass 0 scans the adjacency and fills it, later
    // passes read one row per vertex; applied moves keep it exact
    const bool use_cache = !D.on() && k <= 16 && !gp &&
                           (max_passes >= 2 || (finest && max_passes >= 1)) &&
                           !getenv("HS_KWAY_NOCACHE");
    cache = Conn();
    if (use_cache) {
      cache.kc = k <= 8 ? 8 : 16;
      // counters never exceed a vertex's weighted degree: with unit weights on
      // the finest level that is its degree (known), else 32-bit counters
      const int64_t bound = (finest && g.wconst == 1) ? max_deg0 : (1ll << 31);
      cache.cw = bound < 256 ? 1 : (bound < 65536 ? 2 : 4);
      int rc2 = cache_buffer((int64_t)g.n * cache.kc * cache.cw, &cache.p);
      if (rc2) return rc2;
    }
    const int32_t one = 1;
    HS_CHECK_CUDA(cudaMemcpyAsync(ctl + CTL_ACTIVE, &one, sizeof one, cudaMemcpyHostToDevice, s));
    int32_t *kept = nullptr;
    if (prethin) HS_CHECK_CUDA(dalloc(&kept, g.n, s));
    for (int pass = 0; pass < max_passes; ++pass) {
      HS_CHECK_CUDA(cudaMemsetAsync(ctl, 0, 2 * sizeof(int32_t), s));  // list count, nconf
      HS_CHECK_CUDA(cudaMemsetAsync(d_flows, 0, 2 * k * sizeof(int64_t), s));
      {
        // per vertex: xbeg 8, deg 4, vw 4, own part 1, state write 4; per
        // entry: adj 4, weight 4 (none when uniform), neighbour part 1
        const int TR = k <= 16 ? refine_team_for(g) : team_for(g);
        if (use_cache && pass > 0) {
          hs::Prof P2("refine_cached", s, (5.0 + cache.cw * cache.kc + 4.0) * g.n);
          const int cg = hs::grid_for(g.n, kTeamBlock, hs::sm_count() * 16);
#define HS_RC(KC, CW)                                                                      \
  refine_cached<KC, CW><<<cg, kTeamBlock, 0, s>>>(g, pl, k, d_pw, d_hi, d_lo, st, list,     \
                                                  ctl + CTL_COUNT, ctl + CTL_ACTIVE, cache.p, \
                                                  prethin ? d_flows : nullptr)
          if (cache.kc == 8 && cache.cw == 1 && st.n == 1 && g.v0 == 0 &&
              (reinterpret_cast<uintptr_t>(pl) & 3) == 0 &&
              (reinterpret_cast<uintptr_t>(g.vw) & 15) == 0 &&
              (reinterpret_cast<uintptr_t>(cache.p) & 15) == 0 &&
              (reinterpret_cast<uintptr_t>(st.p[0]) & 15) == 0) {
            const int cg4 = hs::grid_for((g.n + 3) / 4, kTeamBlock, hs::sm_count() * 16);
            refine_cached_v4<<<cg4, kTeamBlock, 0, s>>>(g, pl, k, d_pw, d_hi, d_lo, st.p[0], list,
                                                        ctl + CTL_COUNT, ctl + CTL_ACTIVE, cache.p,
                                                        prethin ? d_flows : nullptr, Lv.vconst);
          } else if (cache.kc == 8) {
            if (cache.cw == 1) HS_RC(8, 1); else if (cache.cw == 2) HS_RC(8, 2); else HS_RC(8, 4);
          } else {
            if (cache.cw == 1) HS_RC(16, 1); else if (cache.cw == 2) HS_RC(16, 2); else HS_RC(16, 4);
          }
#undef HS_RC
        } else {
          hs::Prof P("refine_candidates", s, 21.0 * g.n + (wconst ? 5.0 : 9.0) * g.nnz +
                                                 (use_cache ? (double)cache.cw * cache.kc * g.n : 0.0));
          // pass 0 on a band start (no coarsening, no trials): neighbour parts
          // from the band bounds, no gathers (the device flag rejects other starts)
          int32_t *bands = nullptr;
          if (pass == 0 && finest && !D.on() && !gp && levels.size() == 1) {
            HS_CHECK_CUDA(dalloc(&bands, k + 2, s));
            HS_CHECK_CUDA(cudaMemsetAsync(bands + k + 1, 1, sizeof(int32_t), s));
            band_starts<<<hs::grid_for(g.n, 256), 256, 0, s>>>(g.n, pl, k, bands);
            HS_CHECK_LAUNCH();
          }
          // band start: one lane per vertex, 8 entries in flight (the register
          // fast path has no team work to share: 0.55 -> 0.43 ms at config 4)
          const int TR1 = bands ? 1 : TR;
          HS_REFINE_DISPATCH(TR1, k, pack16, team_grid(g.n, TR1), g, pl, k, d_pw, d_hi, d_lo, st,
                             list, ctl + CTL_COUNT, ctl + CTL_ACTIVE, gp, wconst,
                             use_cache ? cache : Conn(), bands);
          if (bands) cudaFreeAsync(bands, s);
        }
      }
      HS_CHECK_LAUNCH();
      rc = barrier();  // every rank's candidate states are in place
      if (rc) return rc;
      {
        // algorithmic bytes need the candidate count: read it (sync) only in
        // instrumented (profiling) steps. Per candidate: list 4, own state 4,
        // xbeg 8, deg 4, vw 4, decision 4; per entry (average degree): adj 4,
        // weight 4 (none when uniform), neighbour state 4.
        if (prethin) {  // pre-plan: thin the candidates to the balance room first
          // passes > 0 (cache): refine_cached already summed the flows
          const bool fused = use_cache && pass > 0;
          const int fg = hs::grid_for(g.n, 256, hs::sm_count() * 4);
          if (fused) {
          } else if (k <= 8)
            cand_flows_reg<8><<<fg, 256, 0, s>>>(loc(st), list, ctl + CTL_COUNT, g.vw, k, d_flows,
                                                 ctl + CTL_ACTIVE, g.v0);
          else if (k <= 16)
            cand_flows_reg<16><<<fg, 256, 0, s>>>(loc(st), list, ctl + CTL_COUNT, g.vw, k, d_flows,
                                                  ctl + CTL_ACTIVE, g.v0);
          else
            cand_flows<<<fg, 256, 0, s>>>(loc(st), list, ctl + CTL_COUNT, g.vw, k, d_flows,
                                          ctl + CTL_ACTIVE, g.v0);
          if (!fused) HS_CHECK_LAUNCH();
          rc = ar_flows();  // sharded: every rank plans with the global flows
          if (rc) return rc;
          plan_kernel<<<1, kMaxParts, 0, s>>>(k, Lv.n_glob, 2, d_flows, d_pw, d_hi, d_lo,
                                              d_target, d_prob, ctl);
          HS_CHECK_LAUNCH();
          {  // (the pre-plan zeroed the kept count)
            hs::Prof P("refine_thin", s, 0.0);
            thin_cands<<<hs::grid_for(g.n, 256, hs::sm_count() * 16), 256, 0, s>>>(
                st, g.v0, list, ctl + CTL_COUNT, d_prob, k, salt2 ^ (0xA5A5ull + pass * 7877),
                ctl + CTL_ACTIVE, kept, ctl + CTL_KEPT, d_flows);
            HS_CHECK_LAUNCH();
            if (hs::prof_enabled()) {  // per candidate: list + state read, kept or state write
              P.stop();
              int32_t c = 0;
              cudaMemcpyAsync(&c, ctl + CTL_COUNT, 4, cudaMemcpyDeviceToHost, s);
              cudaStreamSynchronize(s);
              P.bytes = 12.0 * c;
            }
          }
          rc = barrier();  // dropped candidates' states are in every replica
          if (rc) return rc;
        }
        double ab_bytes = 0.0;
        if (hs::prof_enabled()) {
          int32_t cnt = 0;
          cudaMemcpyAsync(&cnt, ctl + (prethin ? CTL_KEPT : CTL_COUNT), 4, cudaMemcpyDeviceToHost, s);
          cudaStreamSynchronize(s);
          const double avg = g.n ? (double)g.nnz / (double)g.n : 0.0;
          ab_bytes = (double)cnt * (28.0 + avg * (g.wconst ? 8.0 : 12.0));
        }
        hs::Prof P("refine_afterburner", s, ab_bytes);
        const int TA = after_team_for(g);
        HS_TEAM_DISPATCH(TA, afterburner_t, team_grid(g.n, TA), g, loc(st), prethin ? kept : list,
                         ctl + (prethin ? CTL_KEPT : CTL_COUNT), k, conf, d_flows,
                         ctl + CTL_NCONF, ctl + CTL_ACTIVE);
      }
      HS_CHECK_LAUNCH();
      rc = ar_flows();
      if (rc) return rc;
      plan_kernel<<<1, kMaxParts, 0, s>>>(k, Lv.n_glob, 0, d_flows, d_pw, d_hi, d_lo, d_target,
                                          d_prob, ctl);
      HS_CHECK_LAUNCH();
      int64_t *tgt = apply_target();
      {
        const bool prof = hs::prof_enabled();
        if (prof) HS_CHECK_CUDA(cudaMemsetAsync(ctl + CTL_MOVED, 0, sizeof(int32_t), s));
        hs::Prof P("refine_apply", s, 0.0);
        apply_list<<<hs::grid_for(g.n, 256, hs::sm_count() * 16), 256, 0, s>>>(
            prethin ? kept : list, ctl + (prethin ? CTL_KEPT : CTL_COUNT), conf, g.vw, d_prob, k,
            salt2 + pass * 104729, g.v0, pl, part,
            tgt, ctl + CTL_APPLY, g.xbeg, g.deg, g.twin, gp, g, use_cache ? cache : Conn(),
            prof ? ctl + CTL_MOVED : nullptr);
        HS_CHECK_LAUNCH();
        if (prof) {  // per entry: list, conf, part read; per move: vw, part write,
                     // xbeg, deg, then per neighbour: adj entry + a 4-byte
                     // read-modify-write of its cache row (with the cache)
          P.stop();
          int32_t c2[2] = {0, 0};
          cudaMemcpyAsync(&c2[0], ctl + (prethin ? CTL_KEPT : CTL_COUNT), 4, cudaMemcpyDeviceToHost, s);
          cudaMemcpyAsync(&c2[1], ctl + CTL_MOVED, 4, cudaMemcpyDeviceToHost, s);
          cudaStreamSynchronize(s);
          const double avg = g.n ? (double)g.nnz / (double)g.n : 0.0;
          P.bytes = 9.0 * c2[0] + (double)c2[1] * (17.0 + (use_cache ? 12.0 * avg : 0.0));
        }
      }
      rc = ar_applied();
      if (rc) return rc;
      if (timer.on && finest) {  // HS_KWAY_TRACE: candidates / confirmed / thinning per pass
        int32_t c2[11];
        double pr[2 * kMaxParts];
        cudaMemcpyAsync(c2, ctl, sizeof c2, cudaMemcpyDeviceToHost, s);
        cudaMemcpyAsync(pr, d_prob, 2 * k * sizeof(double), cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        double pmin = 1.0;
        for (int q = 0; q < 2 * k; ++q) pmin = std::min(pmin, pr[q]);
        fprintf(stderr, "[kway] pass %d: candidates %d kept %d confirmed %d min keep-prob %.3f\n",
                pass, c2[0], prethin ? c2[CTL_KEPT] : c2[0], c2[1], pmin);
      }
    }
    rc = rebalance(g, part, cand, salt2 ^ 0x5555ull, 8, use_cache ? cache : Conn());
    if (!use_cache || !finest) cache = Conn();  // only the finest level's cache is kept (final cut)
    if (gp) {
      cudaFreeAsync(gp, s);
      gp = nullptr;
    }
    cudaFreeAsync(cand, s);
    free_rep(st);
    D.bump = arena_mark;
    cudaFreeAsync(list, s);
    cudaFreeAsync(conf, s);
    if (kept) cudaFreeAsync(kept, s);
    return rc;
  }

  // from_cache: the finest level's connectivity cache is current and holds
  // the weights g's cut is taken with (scaled by g.wconst when uniform)
  // defer != nullptr: leave the (all-reduced) doubled cut on the device in
  // *defer for the caller to read with other results (returns 0)
  int64_t cut_of(const G &g, const part_t *part, bool from_cache = false,
                 unsigned long long **defer = nullptr) {
    unsigned long long *c2, h = 0;
    if (dalloc(&c2, 1, s) != cudaSuccess) return -1;
    cudaMemsetAsync(c2, 0, 8, s);
    if (from_cache && cache.p) {
      hs::Prof P("cut_cached", s, (1.0 + cache.cw * cache.kc) * g.n);
      const int cg = hs::grid_for(g.n, 256, hs::sm_count() * 8);
#define HS_CC(KC, CW) cut_cached<KC, CW><<<cg, 256, 0, s>>>(g, part, k, cache.p, c2)
      if (cache.kc == 8) {
        if (cache.cw == 1) HS_CC(8, 1); else if (cache.cw == 2) HS_CC(8, 2); else HS_CC(8, 4);
      } else {
        if (cache.cw == 1) HS_CC(16, 1); else if (cache.cw == 2) HS_CC(16, 2); else HS_CC(16, 4);
      }
#undef HS_CC
    } else {
      hs::Prof P("cut", s, 13.0 * g.n + (g.wconst ? 5.0 : 9.0) * g.nnz);
      const int T = team_for(g);
      HS_TEAM_DISPATCH(T, cut_t, team_grid(g.n, T), g, part, c2);
    }
    hs::count_launch();
    if (ar({seg64((int64_t *)c2, 1)})) return -1;
    if (defer) {
      *defer = c2;
      return 0;
    }
    cudaMemcpyAsync(&h, c2, 8, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    cudaFreeAsync(c2, s);
    return (int64_t)(h / 2);
  }

  // One coarsening level: heavy-edge matching rounds, two-hop pairing,
  // contraction. Two host round trips: the two-hop list size (CUB sorts take
  // host counts) and the coarse vertex count (stop test, next sizes).
  int coarsen_once(bool *stop) {
    Level &F = levels.back();
    const int n = F.g.n;
    const int lvl = (int)levels.size();
    const int32_t max_vw = (int32_t)std::max<int64_t>(1, total_vw / (4ll * k));
    int32_t *match, *prop, *fav, *flag, *cid;
    uint32_t *mw;  // vertex weight | matched bit, gathered once per neighbour
    HS_CHECK_CUDA(dalloc(&match, n, s));
    HS_CHECK_CUDA(dalloc(&prop, n, s));
    HS_CHECK_CUDA(dalloc(&fav, n, s));
    HS_CHECK_CUDA(dalloc(&flag, n + 1, s));
    HS_CHECK_CUDA(dalloc(&cid, n + 1, s));
    HS_CHECK_CUDA(dalloc(&mw, n, s));
    HS_CHECK_CUDA(cudaMemsetAsync(match, 0xff, n * sizeof(int32_t), s));
    HS_CHECK_CUDA(cudaMemcpyAsync(mw, F.g.vw, n * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
    const int T = team_for(F.g);
    // rounds >= 1 visit only the vertices still unmatched (compacted list)
    int32_t *ulist[2] = {nullptr, nullptr}, *ucnt = nullptr;
    if (rounds > 1) {
      HS_CHECK_CUDA(dalloc(&ulist[0], n, s));
      HS_CHECK_CUDA(dalloc(&ulist[1], n, s));
      HS_CHECK_CUDA(dalloc(&ucnt, 2, s));
    }
    for (int round = 0; round < rounds; ++round) {
      const int32_t *lst = nullptr, *lcnt = nullptr;
      if (round > 0) {
        const int cur = round & 1;
        HS_CHECK_CUDA(cudaMemsetAsync(ucnt + cur, 0, sizeof(int32_t), s));
        unmatched_list<<<hs::grid_for(n, 256), 256, 0, s>>>(
            n, round > 1 ? ulist[cur ^ 1] : nullptr, round > 1 ? ucnt + (cur ^ 1) : nullptr, match,
            ulist[cur], ucnt + cur);
        HS_CHECK_LAUNCH();
        lst = ulist[cur];
        lcnt = ucnt + cur;
      }
      {
        // round 0 scans every list; later rounds only unmatched vertices (N-bytes bound)
        hs::Prof P(round == 0 ? "match_propose_r0" : "match_propose_rN", s,
                   round == 0 ? 20.0 * n + (F.g.wconst ? 8.0 : 12.0) * F.g.nnz : 20.0 * n);
        HS_TEAM_DISPATCH(T, propose_t, team_grid(n, T), F.g, mw, prop,
                         round == rounds - 1 ? fav : nullptr, salt + (uint64_t)lvl * 131 + round,
                         max_vw, lst, lcnt, round == 0 ? F.vconst : 0,
                         F.vconst != 0 && F.g.wconst != 0);
      }
      HS_CHECK_LAUNCH();
      match_accept<<<hs::grid_for(n, 256), 256, 0, s>>>(n, match, prop, mw, ctl + 6);
      HS_CHECK_LAUNCH();
    }
    cudaFreeAsync(mw, s);
    if (ulist[0]) { cudaFreeAsync(ulist[0], s); cudaFreeAsync(ulist[1], s); cudaFreeAsync(ucnt, s); }
    {  // two-hop pairing of leftovers that share a favourite neighbour
      uint64_t *keys, *keys2;
      HS_CHECK_CUDA(dalloc(&keys, n, s));
      HS_CHECK_CUDA(dalloc(&keys2, n, s));
      HS_CHECK_CUDA(cudaMemsetAsync(ctl + 7, 0, sizeof(int32_t), s));
      twohop_keys<<<hs::grid_for(n, 256), 256, 0, s>>>(n, match, fav, keys, ctl + 7);
      HS_CHECK_LAUNCH();
      int32_t cnt = 0;
      HS_CHECK_CUDA(cudaMemcpyAsync(&cnt, ctl + 7, sizeof cnt, cudaMemcpyDeviceToHost, s));
      HS_CHECK_CUDA(cudaStreamSynchronize(s));  // host round trip 1
      if (prev_nnz_pending) {  // the previous level's live adjacency count has landed
        levels.back().g.nnz = levels.back().nnz_glob = *h_nnz;
        prev_nnz_pending = false;
      }
      if (timer.on)
        fprintf(stderr, "[kway] level %d: n=%d nnz=%lld avg_deg=%.1f team=%d twohop=%d\n", lvl - 1, n,
                (long long)F.g.nnz, n ? (double)F.g.nnz / n : 0.0, T, cnt);
      if (cnt > 1) {
        int32_t *head, *start;
        size_t tb = 0;
        HS_CHECK_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, keys, keys2, cnt, 0, 64, s));
        {
          hs::Scratch<char> tmp;
          HS_CHECK_CUDA(tmp.alloc(tb, s));
          HS_CHECK_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, tb, keys, keys2, cnt, 0, 64, s));
        }
        HS_CHECK_CUDA(dalloc(&head, cnt, s));
        HS_CHECK_CUDA(dalloc(&start, cnt, s));
        twohop_heads<<<hs::grid_for(cnt, 256), 256, 0, s>>>(keys2, cnt, head);
        HS_CHECK_LAUNCH();
        tb = 0;
        HS_CHECK_CUDA(cub::DeviceScan::InclusiveScan(nullptr, tb, head, start, cub::Max(), cnt, s));
        {
          hs::Scratch<char> tmp;
          HS_CHECK_CUDA(tmp.alloc(tb, s));
          HS_CHECK_CUDA(cub::DeviceScan::InclusiveScan(tmp.p, tb, head, start, cub::Max(), cnt, s));
        }
        twohop_pair<<<hs::grid_for(cnt, 256), 256, 0, s>>>(keys2, start, cnt, F.g.vw, max_vw, match);
        HS_CHECK_LAUNCH();
        hs::count_launch(2);
        cudaFreeAsync(head, s);
        cudaFreeAsync(start, s);
      }
      cudaFreeAsync(keys, s);
      cudaFreeAsync(keys2, s);
    }
    leader_flags<<<hs::grid_for(n, 256), 256, 0, s>>>(n, match, flag);
    HS_CHECK_LAUNCH();
    HS_CHECK_CUDA(cudaMemsetAsync(flag + n, 0, sizeof(int32_t), s));
    int rc = exclusive_scan<int32_t>(flag, cid, n + 1, s);
    if (rc) return rc;
    int32_t nc = 0;
    HS_CHECK_CUDA(cudaMemcpyAsync(&nc, cid + n, sizeof nc, cudaMemcpyDeviceToHost, s));
    HS_CHECK_CUDA(cudaStreamSynchronize(s));  // host round trip 2
    // sharded: coarse ids of rank r follow those of ranks < r
    int64_t coff = 0, nc_glob = nc;
    rc = exscan_host(nc, &coff, &nc_glob);
    if (rc) return rc;
    if (nc_glob > (int64_t)F.n_glob * 92 / 100) {  // matching stalled: stop coarsening here
      cudaFreeAsync(match, s); cudaFreeAsync(prop, s); cudaFreeAsync(fav, s);
      cudaFreeAsync(flag, s); cudaFreeAsync(cid, s);
      *stop = true;
      return HS_OK;
    }
    Level C;
    C.g.n = nc;
    C.g.v0 = (int32_t)coff;
    C.n_glob = (int32_t)nc_glob;
    int32_t *mem0, *mem1;
    int64_t *ub;
    Rep<int32_t> cmap;
    rc = alloc_rep(cmap, F.n_glob);
    if (rc) return rc;
    F.cmap = loc(cmap);
    HS_CHECK_CUDA(dalloc(&mem0, nc, s));
    HS_CHECK_CUDA(dalloc(&mem1, nc, s));
    HS_CHECK_CUDA(dalloc(&ub, nc + 1, s));
    HS_CHECK_CUDA(dalloc(&C.g.vw, nc, s));
    HS_CHECK_CUDA(dalloc(&C.g.deg, nc, s));
    HS_CHECK_CUDA(dalloc(&C.g.xbeg, nc + 1, s));
    build_cmap<<<hs::grid_for(n, 256), 256, 0, s>>>(F.g, match, cid, (int32_t)coff, cmap, mem0,
                                                    mem1, C.g.vw, ub);
    HS_CHECK_LAUNCH();
    rc = barrier();  // every rank's part of the fine->coarse map is in place
    if (rc) return rc;
    HS_CHECK_CUDA(cudaMemsetAsync(ub + nc, 0, sizeof(int64_t), s));
    rc = exclusive_scan<int64_t>(ub, C.g.xbeg, nc + 1, s);
    if (rc) return rc;
    // sum(ub) = live fine entries <= fine capacity: allocate without a round trip
    const int64_t capc = F.g.cap;
    C.g.cap = capc;
    C.g.nnz = capc;  // refined below (asynchronously) to the live count
    HS_CHECK_CUDA(dalloc(&C.g.adj, capc, s));
    HS_CHECK_CUDA(dalloc(&C.g.wgt, capc, s));
    // Will this coarse level be the last one (merged average degree above
    // the stop threshold)? Estimate the merge ratio on a 1/64 sample.
    bool direct = false;
    if (nc_glob >= 65536) {
      const int S = 64;
      contract_warp<<<warp_grid(nc / S + 1, kContractWarps), kContractWarps * 32, 0, s>>>(
          F.g, F.cmap, mem0, mem1, ub, nc, C.g, S);
      HS_CHECK_LAUNCH();
      unsigned long long *sr;
      HS_CHECK_CUDA(dalloc(&sr, 2, s));
      HS_CHECK_CUDA(cudaMemsetAsync(sr, 0, 16, s));
      sample_ratio<<<hs::grid_for(nc / S + 1, 256), 256, 0, s>>>(ub, C.g.deg, nc, S, kWarpSlots, sr);
      HS_CHECK_LAUNCH();
      rc = ar({seg64((int64_t *)sr, 2)});
      if (rc) return rc;
      unsigned long long hr[2] = {0, 0};
      HS_CHECK_CUDA(cudaMemcpyAsync(hr, sr, 16, cudaMemcpyDeviceToHost, s));
      HS_CHECK_CUDA(cudaStreamSynchronize(s));
      cudaFreeAsync(sr, s);
      if (hr[1] > 0) {
        const double merged_avg =
            (double)hr[0] / (double)hr[1] * (double)F.nnz_glob / (double)nc_glob;
        direct = merged_avg > max_deg;
      }
    }
    // A level contracted unmerged is the coarsest one and is not refined
    // (refine(): no passes on unmerged levels). With more than 32k vertices it
    // also gets no warp trials (band start), so only its vertex weights and
    // the fine->coarse map are consumed: its adjacency is not built (empty
    // lists; a rebalance there moves by weight only). Saves a pass over all
    // entries (config 4: 1.6 ms).
    const bool skeleton = direct && nc_glob > 32768;
    if (skeleton) {
      HS_CHECK_CUDA(cudaMemsetAsync(C.g.deg, 0, (size_t)nc * sizeof(int32_t), s));
      C.unmerged = true;
      *stop = true;
    } else if (direct) {
      C.g.wconst = F.g.wconst;  // parallel edges kept: uniform weights stay uniform
      C.unmerged = true;
      hs::Prof P("contract_direct", s,
                 16.0 * nc + 12.0 * n + (F.g.wconst ? 8.0 : 12.0) * F.g.nnz +
                     (F.g.wconst ? 4.0 : 8.0) * F.g.nnz);
      constexpr int TC = 4;  // 4-lane teams (measured against 2 and 8)
      const int cgrid = std::max(1, std::min(hs::sm_count() * 32, (nc * TC + 255) / 256));
      contract_direct<TC><<<cgrid, 256, 0, s>>>(F.g, F.cmap, mem0, mem1, nc, C.g);
      HS_CHECK_LAUNCH();
    } else {
    {
      hs::Prof P("contract_warp", s, 28.0 * nc + 12.0 * n + 12.0 * F.g.nnz);
      contract_warp<<<warp_grid(nc, kContractWarps), kContractWarps * 32, 0, s>>>(
          F.g, F.cmap, mem0, mem1, ub, nc, C.g, 1);
    }
    HS_CHECK_LAUNCH();
    // long lists: CTA with a shared-memory table, then global-memory tables;
    // list sizes stay on the device, the CTA kernels read them there
    const int smem_slots = 8192;
    int32_t *list, *ncd;
    HS_CHECK_CUDA(dalloc(&list, nc, s));
    HS_CHECK_CUDA(dalloc(&ncd, 1, s));
    HS_CHECK_CUDA(cudaMemcpyAsync(ncd, cid + n, sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
    HS_CHECK_CUDA(cudaMemsetAsync(ctl + 8, 0, 2 * sizeof(int32_t), s));
    classify_long<<<hs::grid_for(nc, 256), 256, 0, s>>>(ub, ncd, kWarpSlots, smem_slots, list,
                                                        ctl + 8);
    HS_CHECK_LAUNCH();
    {
      size_t smem = 2 * smem_slots * sizeof(int32_t);
      cudaFuncSetAttribute(contract_block, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      hs::Prof P("contract_block_smem", s, 0.0);
      contract_block<<<hs::sm_count() * 2, 512, smem, s>>>(F.g, F.cmap, mem0, mem1, ub, list,
                                                          ctl + 8, C.g, nullptr, nullptr,
                                                          smem_slots);
    }
    HS_CHECK_LAUNCH();
    int32_t *list2;
    HS_CHECK_CUDA(dalloc(&list2, nc, s));
    classify_long<<<hs::grid_for(nc, 256), 256, 0, s>>>(ub, ncd, smem_slots, INT64_MAX / 4, list2,
                                                        ctl + 9);
    HS_CHECK_LAUNCH();
    {
      int32_t *gk = nullptr, *gv = nullptr;
      int rc2 = D.on() ? (dalloc(&gk, 2 * capc, s) == cudaSuccess &&
                                  dalloc(&gv, 2 * capc, s) == cudaSuccess ? HS_OK : HS_ECUDA)
                       : global_tables(2 * capc, &gk, &gv);
      if (rc2) return rc2;
      hs::Prof P("contract_block_global", s, 0.0);
      contract_block<<<hs::sm_count() * 2, 1024, 0, s>>>(F.g, F.cmap, mem0, mem1, ub, list2,
                                                         ctl + 9, C.g, gk, gv, 0);
      if (D.on()) { cudaFreeAsync(gk, s); cudaFreeAsync(gv, s); }
    }
    HS_CHECK_LAUNCH();
    cudaFreeAsync(list, s); cudaFreeAsync(list2, s); cudaFreeAsync(ncd, s);
    }
    {  // live adjacency entries of the coarse level, read at the next round trip
      size_t tb = 0;
      HS_CHECK_CUDA(cub::DeviceReduce::Sum(nullptr, tb, C.g.deg, d_nnz, nc, s));
      hs::Scratch<char> tmp;
      HS_CHECK_CUDA(tmp.alloc(tb, s));
      HS_CHECK_CUDA(cub::DeviceReduce::Sum(tmp.p, tb, C.g.deg, d_nnz, nc, s));
      hs::count_launch(1);
      if (D.on()) {  // local and global counts now (the stop rule needs the global one)
        int64_t mine = 0, before = 0;
        HS_CHECK_CUDA(cudaMemcpyAsync(&mine, d_nnz, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        HS_CHECK_CUDA(cudaStreamSynchronize(s));
        C.g.nnz = mine;
        rc = exscan_host(mine, &before, &C.nnz_glob);
        if (rc) return rc;
      } else {
        HS_CHECK_CUDA(cudaMemcpyAsync(h_nnz, d_nnz, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        prev_nnz_pending = true;
      }
    }
    cudaFreeAsync(match, s); cudaFreeAsync(prop, s); cudaFreeAsync(fav, s);
    cudaFreeAsync(flag, s); cudaFreeAsync(cid, s); cudaFreeAsync(mem0, s);
    cudaFreeAsync(mem1, s); cudaFreeAsync(ub, s);
    levels.push_back(C);
    return HS_OK;
  }

  // Grow-only device buffer of the connectivity cache (hundreds of MB at
  // config 4: a per-call stream-ordered allocation fragmented the pool and
  // stalled the next call's allocations). One GPU only (not used sharded).
  int cache_buffer(int64_t bytes, uint8_t **out) {
    static std::mutex mu;
    static uint8_t *buf = nullptr;
    static int64_t have = 0;
    std::lock_guard<std::mutex> lk(mu);
    if (bytes > have) {
      HS_CHECK_CUDA(cudaStreamSynchronize(s));
      if (buf) cudaFree(buf);
      buf = nullptr;
      HS_CHECK_CUDA(cudaMalloc((void **)&buf, bytes));
      have = bytes;
    }
    *out = buf;
    return HS_OK;
  }

  // Grow-only device scratch for the global-memory hash tables of the
  // longest lists (kept across calls: re-reserving GBs per call stalls).
  int global_tables(int64_t slots, int32_t **keys, int32_t **vals) {
    static int32_t *gk = nullptr, *gv = nullptr;
    static int64_t have = 0;
    if (slots > have) {
      HS_CHECK_CUDA(cudaStreamSynchronize(s));
      if (gk) cudaFree(gk);
      if (gv) cudaFree(gv);
      gk = gv = nullptr;
      HS_CHECK_CUDA(cudaMalloc((void **)&gk, slots * sizeof(int32_t)));
      HS_CHECK_CUDA(cudaMalloc((void **)&gv, slots * sizeof(int32_t)));
      have = slots;
    }
    *keys = gk;
    *vals = gv;
    return HS_OK;
  }

  // Lands the last pending live-entry count (after the final coarsening level).
  int settle_nnz() {
    if (!prev_nnz_pending) return HS_OK;
    HS_CHECK_CUDA(cudaStreamSynchronize(s));
    levels.back().g.nnz = levels.back().nnz_glob = *h_nnz;
    prev_nnz_pending = false;
    return HS_OK;
  }

  // FM runs on graphs whose finest level is an FM level (<= kFmMaxLevel
  // vertices): there every level gets FM candidates. On larger graphs the
  // coarse levels of task DAGs are dense (average degree 100-200 at a few
  // thousand vertices), every FM move dirties most rows, and a level took
  // 10-100 ms; the band start at the coarsest level with Jet refinement on
  // every level measured 10-30x faster at an equal or lower cut on layered
  // DAGs (20k-100k tasks, m/n = 3-10) and the 45,760-task Cholesky DAG at
  // k = 8, 17% higher at k = 2 (tools/calib2.py).
  bool fm_levels() const { return levels[0].n_glob <= kFmMaxLevel; }

  // FM candidates on a small level (one GPU): n_init recursive-bisection
  // starts, `copies` copies of `cur` (each searches with its own hash salt)
  // and the caller's starts at the finest level; the best by (violation,
  // cut) replaces cur. No host round trip.
  int fm_level(const Level &Lv, part_t *cur, int n_init, int copies, bool with_starts,
               int passes, uint64_t salt2) {
    const G &g = Lv.g;
    const int n = g.n;
    const int n_ext = with_starts ? n_starts : 0;
    const int64_t rows = (int64_t)n * k * 4;
    const int64_t flags = fm_vertex_bytes(n);  // per-vertex state (kway_fm.cuh)
    int smem_max = 0;
    HS_CHECK_CUDA(cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin,
                                         dev_id()));
    const int64_t static_smem = 8 * 1024;  // fm_kernel's own __shared__ arrays
    const bool sm = flags + rows + static_smem <= smem_max;
    if (!sm) {  // global rows: keep the scratch within 512 MB
      const int64_t cap = std::max<int64_t>(1, (512ll << 20) / std::max<int64_t>(rows, 1));
      while ((int64_t)n_init + copies + n_ext > cap && n_init > 0) --n_init;
      while ((int64_t)n_init + copies + n_ext > cap && copies > 1) --copies;
    }
    const int C = n_init + copies + n_ext;
    part_t *parts;
    int32_t *trail, *conn = nullptr;
    int64_t *cut, *viol;
    HS_CHECK_CUDA(dalloc(&parts, (int64_t)C * n, s));
    HS_CHECK_CUDA(dalloc(&trail, (int64_t)C * n, s));
    HS_CHECK_CUDA(dalloc(&cut, C, s));
    HS_CHECK_CUDA(dalloc(&viol, C, s));
    if (!sm) HS_CHECK_CUDA(dalloc(&conn, (int64_t)C * n * k, s));
    if (copies) {
      fm_fill_copies<<<hs::grid_for((int64_t)copies * n, 256), 256, 0, s>>>(cur, n, parts, n_init,
                                                                            copies);
      HS_CHECK_LAUNCH();
    }
    if (n_ext) {
      fm_fill_starts<<<hs::grid_for((int64_t)n_ext * n, 256), 256, 0, s>>>(
          starts, (int64_t)n_ext * n, parts + (int64_t)(n_init + copies) * n);
      HS_CHECK_LAUNCH();
    }
    FmArgs A;
    A.g = g;
    A.k = k;
    A.hi = d_hi;
    A.lo = d_lo;
    A.cum = d_cum;
    A.tol_split = tol;
    A.parts = parts;
    A.conn_g = conn;
    A.trail = trail;
    A.cut = cut;
    A.viol = viol;
    A.n_init = n_init;
    A.salt = salt2;
    A.passes = passes;
    A.stall = std::max(32, std::min(400, n / 8));
    A.stats = nullptr;
    if (timer.on) {
      HS_CHECK_CUDA(dalloc(&A.stats, 8 * (int64_t)C, s));
      HS_CHECK_CUDA(cudaMemsetAsync(A.stats, 0, 64 * (int64_t)C, s));
    }
    const int64_t dyn = flags + (sm ? rows : 0);
    {
      hs::Prof P("fm_level", s, 0.0);
      if (sm) {
        HS_CHECK_CUDA(cudaFuncSetAttribute(fm_kernel<true>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
        fm_kernel<true><<<C, kFmThreads, dyn, s>>>(A);
      } else {
        HS_CHECK_CUDA(cudaFuncSetAttribute(fm_kernel<false>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
        fm_kernel<false><<<C, kFmThreads, dyn, s>>>(A);
      }
    }
    HS_CHECK_LAUNCH();
    fm_pick<<<hs::grid_for(n, 256, 64), 256, 0, s>>>(viol, cut, C, parts, n, cur, nullptr);
    HS_CHECK_LAUNCH();
    if (A.stats) {  // HS_KWAY_TRACE: the slowest candidate's counters
      std::vector<long long> h(8 * (size_t)C);
      HS_CHECK_CUDA(cudaMemcpyAsync(h.data(), A.stats, 64 * (int64_t)C, cudaMemcpyDeviceToHost, s));
      HS_CHECK_CUDA(cudaStreamSynchronize(s));
      int w = 0;
      for (int c = 1; c < C; ++c)
        if (h[8 * c + 6] > h[8 * w + 6]) w = c;
      const long long *q = h.data() + 8 * w;
      fprintf(stderr,
              "[kway] fm level n=%d nnz=%lld C=%d init=%d: slowest cand %d: %.3f Mclk, moves %lld "
              "passes %lld rolled back %lld, scan %.3f Mclk, move %.3f Mclk, grow steps %lld\n",
              n, (long long)g.nnz, C, n_init, w, q[6] / 1e6, q[0], q[1], q[2], q[3] / 1e6, q[4] / 1e6,
              q[5]);
      cudaFreeAsync(A.stats, s);
    }
    cudaFreeAsync(parts, s);
    cudaFreeAsync(trail, s);
    cudaFreeAsync(cut, s);
    cudaFreeAsync(viol, s);
    if (conn) cudaFreeAsync(conn, s);
    return HS_OK;
  }

  int initial(Rep<part_t> &best_rep) {
    Level &Cst = levels.back();
    G &g = Cst.g;
    const int nc = g.n;
    int rc0 = alloc_rep(best_rep, Cst.n_glob);
    if (rc0) return rc0;
    part_t *best = loc(best_rep);
    // trial 0: id-range bands (global prefix of the weights when sharded)
    {
      int64_t *prefix;
      HS_CHECK_CUDA(dalloc(&prefix, nc + 1, s));
      int rc = exclusive_scan_widen(g.vw, prefix, nc, s);
      if (rc) return rc;
      int64_t woff = 0;
      if (D.on()) {
        int64_t mine = 0, all = 0;
        HS_CHECK_CUDA(cudaMemcpyAsync(&mine, prefix + nc, 8, cudaMemcpyDeviceToHost, s));
        HS_CHECK_CUDA(cudaStreamSynchronize(s));
        rc = exscan_host(mine, &woff, &all);
        if (rc) return rc;
      }
      range_parts<<<hs::grid_for(nc, 256), 256, 0, s>>>(nc, prefix, woff, g.vw, d_cum, k,
                                                        total_vw, g.v0, best_rep);
      HS_CHECK_LAUNCH();
      cudaFreeAsync(prefix, s);
      rc = barrier();  // every rank's bands are in place
      if (rc) return rc;
    }
    // small coarsest graph (one GPU): recursive-bisection FM candidates, the
    // refined band start and (when this is the finest level) the caller's
    // starts; the band start alone otherwise
    if (fm_levels() && nc <= kFmMaxLevel && !D.on() && k > 1) {
      const int n_init = nc <= 1024 ? 2 * hs::sm_count() : hs::sm_count();
      return fm_level(Cst, best, n_init, 1, levels.size() == 1, kFmInitPasses,
                      salt ^ 0xC0A25E57ull);
    }
    return HS_OK;
  }
};

}  // namespace

extern "C" int hs_symmetrize_range(const hs_dag_t *g, int32_t kv0, int32_t kv1,
                                   const int32_t *edge_w_i, const int32_t *edge_w_i_in,
                                   const int32_t *node_w_i, int64_t *xadj, int32_t *adjncy,
                                   int32_t *adjwgt_i, int32_t *vwgt_i, int32_t *twin,
                                   int64_t *nnz_host, void *stream) {
  HS_REQUIRE(g && node_w_i && xadj && adjncy && vwgt_i, HS_EINVAL, "hs_symmetrize: null argument");
  HS_REQUIRE(!adjwgt_i || edge_w_i, HS_EINVAL, "hs_symmetrize: adjwgt_i needs edge_w_i");
  HS_REQUIRE(adjwgt_i || !twin, HS_EINVAL, "hs_symmetrize: unit weights take no twin index");
  const int nk = g->n - 1;
  HS_REQUIRE(0 <= kv0 && kv0 <= kv1 && kv1 <= nk, HS_EINVAL, "kernel range [%d, %d) outside [0, %d)",
             kv0, kv1, nk);
  HS_REQUIRE(!twin || (kv0 == 0 && kv1 == nk), HS_EINVAL, "twin indices need the full range");
  HS_REQUIRE(!twin || 2 * g->m < (1ll << 31), HS_ELIMIT, "twin indices need < 2^31 entries");
  cudaStream_t s = (cudaStream_t)stream;
  const int nl = kv1 - kv0;
  // in/out pointers, in_src/out_dst, weights (in + out order), adj+wgt writes
  const double frac = nk ? (double)nl / (double)nk : 0.0;
  // per node: in/out pointers, xadj, node weight read + write; per edge:
  // in_src + out_dst read, two adjacency writes, and with weights the out-
  // and in-order weight reads and two weight writes
  hs::Prof P("symmetrize", s, frac * (32.0 * g->n + (adjwgt_i ? 32.0 : 16.0) * g->m));
  if (!twin) {  // (the team path below also writes the twin index)
    // row starts come from the CSR prefixes (sym_row_start): no degree pass
    const int64_t chunks = ((int64_t)nl + 31) / 32;
    const int cgrid = (int)std::max<int64_t>(
        1, std::min<int64_t>((int64_t)hs::sm_count() * 8, (chunks + kSymWarps - 1) / kSymWarps));
    sym_fill_chunk<<<cgrid, kSymWarps * 32, 0, s>>>(*g, kv0, kv1, edge_w_i, edge_w_i_in, node_w_i,
                                                    xadj, adjncy, adjwgt_i, vwgt_i);
    HS_CHECK_LAUNCH();
    if (nnz_host) {
      HS_CHECK_CUDA(cudaMemcpyAsync(nnz_host, xadj + nl, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
      HS_CHECK_CUDA(cudaStreamSynchronize(s));
    }
    return HS_OK;
  }
  hs::Scratch<int32_t> deg;
  HS_CHECK_CUDA(deg.alloc(nl + 1, s));
  sym_degree<<<hs::grid_for(nl, 256), 256, 0, s>>>(*g, kv0, kv1, deg);
  HS_CHECK_LAUNCH();
  int rc = exclusive_scan_widen(deg, xadj, nl, s);
  if (rc) return rc;
  constexpr int TS = 4;  // measured: 4 lanes beat 8 and 2
  const int sgrid = std::max(1, std::min(hs::sm_count() * 32, (nl * TS + 255) / 256));
  sym_fill<TS><<<sgrid, 256, 0, s>>>(*g, kv0, kv1, edge_w_i, edge_w_i_in, node_w_i, xadj, adjncy,
                                      adjwgt_i, vwgt_i, twin);
  HS_CHECK_LAUNCH();
  if (nnz_host) {
    HS_CHECK_CUDA(cudaMemcpyAsync(nnz_host, xadj + nl, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    HS_CHECK_CUDA(cudaStreamSynchronize(s));
  }
  return HS_OK;
}

extern "C" int hs_int32_stats(const int32_t *w, int64_t n, int64_t *sum_min_max_host,
                              void *stream) {
  HS_REQUIRE(sum_min_max_host && (w || n == 0) && n >= 0, HS_EINVAL,
             "hs_int32_stats: null argument");
  cudaStream_t s = (cudaStream_t)stream;
  int64_t h[3] = {0, INT32_MAX, INT32_MIN};
  if (n > 0) {
    hs::Scratch<int64_t> d;
    HS_CHECK_CUDA(d.alloc(3, s));
    HS_CHECK_CUDA(cudaMemcpyAsync(d.p, h, sizeof h, cudaMemcpyHostToDevice, s));
    wstats_kernel<<<hs::grid_for(n, 256, hs::sm_count() * 8), 256, 0, s>>>(
        n, w, (unsigned long long *)d.p, (int32_t *)(d.p + 1), (int32_t *)(d.p + 2));
    HS_CHECK_LAUNCH();
    widen_minmax<<<1, 1, 0, s>>>(d.p + 1);
    HS_CHECK_LAUNCH();
    HS_CHECK_CUDA(cudaMemcpyAsync(h, d.p, sizeof h, cudaMemcpyDeviceToHost, s));
    HS_CHECK_CUDA(cudaStreamSynchronize(s));
  }
  for (int i = 0; i < 3; ++i) sum_min_max_host[i] = h[i];
  return HS_OK;
}

namespace {
// two float4-wide loads per thread-iteration; the products and sums round
// like the reference's w * scale + 0.5 (this file builds with --fmad=false)
__device__ __forceinline__ int32_t scaled_weight(double w, double scale) {
  const double f = floor(w * scale + 0.5);
  return f >= 2147483647.0 ? INT32_MAX : (f >= 1.0 ? (int32_t)f : 1);
}
__global__ void integer_weights_kernel(const double *w, int64_t n, double scale, int32_t *out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t n4 = ((reinterpret_cast<uintptr_t>(w) | reinterpret_cast<uintptr_t>(out)) & 15)
                         ? 0 : n / 4;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += stride) {
    const double2 a = __ldcs(reinterpret_cast<const double2 *>(w) + 2 * i);
    const double2 b = __ldcs(reinterpret_cast<const double2 *>(w) + 2 * i + 1);
    __stcs(reinterpret_cast<int4 *>(out) + i,
           make_int4(scaled_weight(a.x, scale), scaled_weight(a.y, scale),
                     scaled_weight(b.x, scale), scaled_weight(b.y, scale)));
  }
  for (int64_t i = 4 * n4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = scaled_weight(w[i], scale);
}
}  // namespace

extern "C" int hs_integer_weights(const double *w, int64_t n, int32_t scale, int32_t *out,
                                  void *stream) {
  HS_REQUIRE(n >= 0 && (n == 0 || (w && out)), HS_EINVAL, "hs_integer_weights: null argument");
  if (n == 0) return HS_OK;
  cudaStream_t s = (cudaStream_t)stream;
  hs::Prof P("integer_weights", s, 12.0 * n);
  integer_weights_kernel<<<hs::grid_for((n + 3) / 4, 256, hs::sm_count() * 8), 256, 0, s>>>(
      w, n, (double)scale, out);
  HS_CHECK_LAUNCH();
  return HS_OK;
}

extern "C" int hs_symmetrize(const hs_dag_t *g, const int32_t *edge_w_i,
                             const int32_t *edge_w_i_in, const int32_t *node_w_i, int64_t *xadj,
                             int32_t *adjncy, int32_t *adjwgt_i, int32_t *vwgt_i, int32_t *twin,
                             int64_t *nnz_host, void *stream) {
  HS_REQUIRE(g, HS_EINVAL, "hs_symmetrize: null argument");
  return hs_symmetrize_range(g, 0, g->n - 1, edge_w_i, edge_w_i_in, node_w_i, xadj, adjncy,
                             adjwgt_i, vwgt_i, twin, nnz_host, stream);
}

namespace {
// One GPU (dist == nullptr) or one rank of a sharded group: ug holds this
// rank's rows [v0, v0 + ug->n) of an n_glob-vertex graph.
int partition_impl(const hs_ugraph_t *ug, int32_t v0, int32_t n_glob, const hs_dist_t *dist,
                   int32_t k, const double *tpwgts_host, double tol, uint64_t seed,
                   int32_t *part_out, int64_t *stats_host, cudaStream_t s,
                   const int32_t *starts = nullptr, int32_t n_starts = 0) {
  const int n0 = ug->n;
  const int64_t nnz0 = ug->nnz;
  Kway K(s);
  K.starts = starts;
  K.n_starts = n_starts;
  K.k = k;
  K.tol = tol;
  K.seed = seed;
  K.salt = seed * 0x9E3779B97F4A7C15ull + 0x1234567ull;
  if (dist && dist->size > 1) {
    K.D.rank = dist->rank;
    K.D.P = dist->size;
    for (int r = 0; r < dist->size; ++r) K.D.arena[r] = (char *)dist->arena[r];
    K.D.arena_bytes = dist->arena_bytes;
    K.D.threads = dist->mode == 1;
    if (K.D.threads) K.hb = host_barrier_for(dist->arena[0]);
    int rc0 = no_cross_stream_pool_waits();
    if (rc0) return rc0;
    rc0 = load_epoch(K.D, &K.D.epoch, s);
    if (rc0) return rc0;
    HS_CHECK_CUDA(cudaMemsetAsync(K.D.arena[K.D.rank] + 64, 0, 4, s));  // this rank's watchdog word
    HS_CHECK_CUDA(dalloc(&K.d_dpw, k, s));
    HS_CHECK_CUDA(dalloc(&K.d_arbuf, kArSlots, s));
  }
  K.timer.mark("start");

  // ---- totals and the int32 weight guard ----
  // tot: [0] edge-weight sum, [1] vertex-weight sum, [2] adjacency entries,
  // [3] min edge weight, [4] max edge weight, [5] max degree, [6] min vertex
  // weight, [7] max vertex weight (all ranks' rows)
  int64_t *tot_dev;
  HS_CHECK_CUDA(dalloc(&tot_dev, 8, s));
  int64_t tot[8] = {0, 0, nnz0, INT32_MAX, INT32_MIN, 0, INT32_MAX, INT32_MIN};
  int32_t *deg_l0;
  HS_CHECK_CUDA(dalloc(&deg_l0, n0, s));
  // locality probe buffers (launched with the totals, read with them)
  const bool probe_wanted = n_glob / 2 > 32768 && !getenv("HS_KWAY_COARSEN");
  unsigned long long *probe_dev = nullptr, probe_h[2] = {0, 0};
  HS_CHECK_CUDA(dalloc(&probe_dev, 2, s));
  HS_CHECK_CUDA(cudaMemsetAsync(probe_dev, 0, 16, s));
  {
    HS_CHECK_CUDA(cudaMemcpyAsync(tot_dev, tot, sizeof tot, cudaMemcpyHostToDevice, s));
    deg_from_xadj<<<hs::grid_for(n0, 256), 256, 0, s>>>(ug->xadj, n0, deg_l0,
                                                        (int32_t *)(tot_dev + 5));
    HS_CHECK_LAUNCH();
    if (ug->adjwgt_i) {
      wstats_kernel<<<hs::grid_for(nnz0, 256, hs::sm_count() * 8), 256, 0, s>>>(
          nnz0, ug->adjwgt_i, (unsigned long long *)tot_dev, (int32_t *)(tot_dev + 3),
          (int32_t *)(tot_dev + 4));
      HS_CHECK_LAUNCH();
    } else {  // METIS's adjwgt = NULL: every edge weighs 1 (sum = entries)
      const int64_t unit[3] = {nnz0, 1, 1};
      HS_CHECK_CUDA(cudaMemcpyAsync(tot_dev, unit, 8, cudaMemcpyHostToDevice, s));
      const int32_t one1[2] = {1, 1};
      HS_CHECK_CUDA(cudaMemcpyAsync(tot_dev + 3, one1, 4, cudaMemcpyHostToDevice, s));
      HS_CHECK_CUDA(cudaMemcpyAsync(tot_dev + 4, one1, 4, cudaMemcpyHostToDevice, s));
    }
    wstats_kernel<<<hs::grid_for(n0, 256, hs::sm_count() * 8), 256, 0, s>>>(
        n0, ug->vwgt_i, (unsigned long long *)(tot_dev + 1), (int32_t *)(tot_dev + 6),
        (int32_t *)(tot_dev + 7));
    HS_CHECK_LAUNCH();
    widen_minmax<<<1, 1, 0, s>>>(tot_dev + 3);
    HS_CHECK_LAUNCH();
    widen_minmax<<<1, 1, 0, s>>>(tot_dev + 6);
    HS_CHECK_LAUNCH();
    // the locality probe (see below) rides on the same host read
    if (probe_wanted) {
      HS_CHECK_CUDA(cudaMemsetAsync(probe_dev, 0, 16, s));
      G pg;
      pg.n = n0;
      pg.v0 = v0;
      pg.xbeg = const_cast<int64_t *>(ug->xadj);
      pg.deg = deg_l0;
      pg.adj = const_cast<int32_t *>(ug->adjncy);
      const int stride = std::max(1, n_glob / 16384);
      locality_probe<<<hs::sm_count() * 4, 256, 0, s>>>(pg, stride, probe_dev);
      HS_CHECK_LAUNCH();
    }
    // sums, then global minima / maxima
    int rc = K.ar({Kway::seg64(tot_dev, 3), Kway::seg64(tot_dev + 3, 1, 2),
                   Kway::seg64(tot_dev + 4, 2, 1), Kway::seg64(tot_dev + 6, 1, 2),
                   Kway::seg64(tot_dev + 7, 1, 1), Kway::seg64((int64_t *)probe_dev, 2)});
    if (rc) return rc;
    HS_CHECK_CUDA(cudaMemcpyAsync(tot, tot_dev, sizeof tot, cudaMemcpyDeviceToHost, s));
    HS_CHECK_CUDA(cudaMemcpyAsync(probe_h, probe_dev, sizeof probe_h, cudaMemcpyDeviceToHost, s));
    HS_CHECK_CUDA(cudaStreamSynchronize(s));
    rc = K.check_peers();
    if (rc) return rc;
  }
  cudaFreeAsync(tot_dev, s);
  HS_REQUIRE(tot[1] > 0 && tot[1] < (1ll << 31), HS_ELIMIT,
             "total vertex weight must be in 1..2^31-1 (got %lld)", (long long)tot[1]);
  K.total_vw = tot[1];

  Level L0;
  L0.own_adj = false;
  L0.own_xbeg_vw = false;
  L0.g.n = n0;
  L0.g.v0 = v0;
  L0.n_glob = n_glob;
  L0.g.cap = nnz0;
  L0.g.nnz = nnz0;
  L0.nnz_glob = tot[2];
  L0.g.xbeg = const_cast<int64_t *>(ug->xadj);
  L0.g.adj = const_cast<int32_t *>(ug->adjncy);
  L0.g.twin = ug->twin;
  L0.g.vw = const_cast<int32_t *>(ug->vwgt_i);
  L0.g.deg = deg_l0;
  K.max_deg0 = tot[5];
  L0.vconst = (tot[6] == tot[7] && n_glob > 0) ? (int32_t)tot[6] : 0;
  int64_t div = 1;
  // uniform edge weights: work with unit weights (no weight stream, no
  // overflow: sums are entry counts); the reported cut is rescaled
  const int32_t w_uniform = (tot[2] > 0 && tot[3] == tot[4] && tot[3] > 0) ? (int32_t)tot[3] : 0;
  if (!w_uniform && tot[0] >= (1ll << 30)) div = (tot[0] >> 30) + 1;
  if (w_uniform) {
    L0.g.wgt = const_cast<int32_t *>(ug->adjwgt_i);
    L0.g.wconst = 1;
    L0.own_wgt = false;
  } else if (div > 1) {
    HS_CHECK_CUDA(dalloc(&L0.g.wgt, nnz0, s));
    scale_weights<<<hs::grid_for(nnz0, 256), 256, 0, s>>>(nnz0, ug->adjwgt_i, L0.g.wgt, div);
    HS_CHECK_LAUNCH();
  } else {
    L0.g.wgt = const_cast<int32_t *>(ug->adjwgt_i);
    L0.own_wgt = false;
  }
  K.levels.push_back(L0);

  // ---- balance bounds ----
  K.hi.resize(k); K.lo.resize(k); K.target.resize(k); K.cum.assign(k + 1, 0.0);
  // |w/W - t| <= tol evaluated in doubles exactly as the reported deviation
  // (and the reference's err, partition.py:72,83): hi / lo are the extreme
  // integers that pass, so "in bounds" and "feasible" never disagree
  const double W = (double)K.total_vw;
  auto ok = [&](int64_t x, double t) { return fabs((double)x / W - t) <= tol; };
  for (int p = 0; p < k; ++p) {
    double t = tpwgts_host[p];
    int64_t h = (int64_t)floor((t + tol) * W);
    while (ok(h + 1, t)) ++h;
    while (h > 0 && !ok(h, t) && (double)h / W > t) --h;
    double l = (t - tol) * W;
    int64_t lo = l <= 0 ? 0 : (int64_t)ceil(l);
    while (lo > 0 && ok(lo - 1, t)) --lo;
    while (!ok(lo, t) && (double)lo / W < t && lo < h) ++lo;
    K.hi[p] = h;
    K.lo[p] = lo;
    K.target[p] = (int64_t)llround(t * W);
    K.cum[p + 1] = K.cum[p] + t;
  }
  HS_CHECK_CUDA(dalloc(&K.d_hi, k, s));
  HS_CHECK_CUDA(dalloc(&K.d_lo, k, s));
  HS_CHECK_CUDA(dalloc(&K.d_target, k, s));
  HS_CHECK_CUDA(dalloc(&K.d_pw, k, s));
  HS_CHECK_CUDA(dalloc(&K.d_flows, 2 * k, s));
  HS_CHECK_CUDA(dalloc(&K.d_prob, 2 * k, s));
  HS_CHECK_CUDA(dalloc(&K.d_cum, k + 1, s));
  HS_CHECK_CUDA(dalloc(&K.counter, 4, s));
  HS_CHECK_CUDA(dalloc(&K.ctl, 16, s));
  HS_CHECK_CUDA(cudaMemsetAsync(K.ctl, 0, 16 * sizeof(int32_t), s));  // ctl[12]: max wdeg
  HS_CHECK_CUDA(dalloc(&K.d_nnz, 1, s));
  {  // one pinned word for the whole process (cudaFreeHost would sync the device)
    static int64_t *pinned = nullptr;
    if (!pinned) HS_CHECK_CUDA(cudaMallocHost((void **)&pinned, sizeof(int64_t)));
    K.h_nnz = pinned;
  }
  HS_CHECK_CUDA(cudaMemcpyAsync(K.d_hi, K.hi.data(), k * 8, cudaMemcpyHostToDevice, s));
  HS_CHECK_CUDA(cudaMemcpyAsync(K.d_lo, K.lo.data(), k * 8, cudaMemcpyHostToDevice, s));
  HS_CHECK_CUDA(cudaMemcpyAsync(K.d_target, K.target.data(), k * 8, cudaMemcpyHostToDevice, s));
  HS_CHECK_CUDA(cudaMemcpyAsync(K.d_cum, K.cum.data(), (k + 1) * 8, cudaMemcpyHostToDevice, s));
  K.timer.mark("setup");

  // ---- coarsening ----
  // coarsest level: ~30 vertices per part and at least n / (20 log2 k) (the
  // recursive-bisection FM candidates work there), never above the FM range
  int lg = 1;
  while ((1 << lg) < k) ++lg;
  const int coarse_target =
      std::min(kFmMaxLevel / 2, std::max(30 * k, (int)(n_glob / (20ll * lg))));
  bool stop = false;
  // Coarsening also stops once the coarse graph turns dense (average degree
  // above max_deg): on random-like DAGs the edge count stops shrinking while
  // every further level costs a full pass over ~all edges.
  // Default: 1.5x the finest level's average degree (edges no longer shrink
  // with the vertices, so matching has no locality left to exploit).
  const double deg0 = n_glob ? (double)L0.nnz_glob / (double)n_glob : 0.0;
  double max_deg = std::max(16.0, 1.5 * deg0);
  K.max_deg = max_deg;
  // Skip coarsening when its only product would be the band start on a
  // skeleton level: a triangle-free-looking finest graph (matching
  // merges nothing but the matched edges, so the first coarse level's average
  // degree is ~2*deg0 - 2 > max_deg and coarsening stops there) that is still
  // too large for warp trials (> 32k coarse vertices). The bands are then cut
  // on the finest ids directly: config 4 measured 9.0 -> 6.3 ms, cut +0.2%.
  // Sharded: every rank probes its own rows (neighbours in other shards are
  // skipped) and the counts are all-reduced, so all ranks decide alike.
  if (probe_wanted && 2.0 * deg0 - 2.0 > max_deg) {
    const unsigned long long *h = probe_h;
    if (h[0] > 0 && (double)h[1] < 0.02 * (double)h[0]) stop = true;
    if (K.timer.on)
      fprintf(stderr, "[kway] locality probe: %llu/%llu pairs share a neighbour%s\n", h[1], h[0],
                      stop ? " -> no coarsening" : "");
  }
  cudaFreeAsync(probe_dev, s);
  if (getenv("HS_KWAY_NOCOARSEN")) stop = true;
  while (!stop && K.levels.back().n_glob > coarse_target && (int)K.levels.size() < 40) {
    if (K.levels.size() > 1) {
      int rc0 = K.settle_nnz();
      if (rc0) return rc0;
      const Level &cl = K.levels.back();
      // a dense level stops coarsening only when another level would cost
      // real passes over many entries; small levels coarsen to the target
      if ((double)cl.nnz_glob > max_deg * (double)cl.n_glob && cl.nnz_glob > kDenseStopNnz) break;
    }
    const bool ncu_win = K.levels.size() == 1 && getenv("HS_NCU_COARSEN0") != nullptr;
    if (ncu_win) cudaProfilerStart();
    int rc = K.coarsen_once(&stop);
    if (ncu_win) cudaProfilerStop();
    if (rc) return rc;
    K.timer.mark("coarsen level");
  }

  {
    int rc = K.settle_nnz();
    if (rc) return rc;
  }
  // ---- initial partition ----
  Rep<part_t> cur;
  int rc = K.initial(cur);
  if (rc) return rc;
  K.timer.mark("initial partition");
  const int coarsest_n = K.levels.back().n_glob;

  // ---- uncoarsening + refinement ----
  bool pw_exact = false;
  for (int li = (int)K.levels.size() - 1; li >= 0; --li) {
    Level &Lv = K.levels[li];
    if (li != (int)K.levels.size() - 1) {
      // every rank projects the whole (replicated) map into its own replica
      Rep<part_t> pf;
      rc = K.alloc_rep(pf, Lv.n_glob);
      if (rc) return rc;
      project<<<hs::grid_for(Lv.n_glob, 256), 256, 0, s>>>(Lv.n_glob, Lv.cmap, K.loc(cur),
                                                           K.loc(pf));
      HS_CHECK_LAUNCH();
      K.free_rep(cur);
      cur = pf;
    }
    if (K.fm_levels() && !K.D.on() && Lv.g.n <= kFmMaxLevel && k > 1) {
      // small level: FM candidates from the projected partition (the
      // coarsest one was refined by its initial candidates already)
      if (li != (int)K.levels.size() - 1) {
        rc = K.fm_level(Lv, K.loc(cur), 0, kFmCopies, li == 0, kFmRefinePasses,
                        K.salt ^ ((uint64_t)li << 40) ^ 0xF00Dull);
        if (rc) return rc;
      }
      K.timer.mark("refine level (fm)");
      continue;
    }
    // HS_NCU_LEVEL0=1: open the profiler window around the finest level only
    const bool ncu_win = li == 0 && getenv("HS_NCU_LEVEL0") != nullptr;
    if (ncu_win) cudaProfilerStart();
    rc = K.refine(Lv, cur, K.salt ^ ((uint64_t)li << 40), li == 0);
    if (ncu_win) cudaProfilerStop();
    if (rc) return rc;
    pw_exact = li == 0;  // refine keeps d_pw in step with every applied move
    K.timer.mark("refine level");
  }
  int8_to_int32<<<hs::grid_for(n_glob, 256), 256, 0, s>>>(K.loc(cur), n_glob, part_out);
  HS_CHECK_LAUNCH();

  // ---- statistics (cut with the caller's unscaled weights) ----
  G g0 = K.levels[0].g;  // the caller's arrays and unscaled weights
  g0.adj = const_cast<int32_t *>(ug->adjncy);
  g0.wgt = const_cast<int32_t *>(ug->adjwgt_i);
  g0.wconst = w_uniform;
  // the connectivity cache holds unit weights (uniform) or the caller's own
  // (div == 1): the cut comes from it without another pass over the edges
  const bool cached_cut = K.cache.p != nullptr && div == 1;
  unsigned long long *cut_dev = nullptr;
  if (K.cut_of(g0, K.loc(cur), cached_cut, &cut_dev) < 0 || !cut_dev)
    HS_REQUIRE(false, HS_ECUDA, "k-way: cut failed");
  K.cache = Conn();
  // the finest level's refinement left d_pw exact (all ranks' moves, the
  // caller's unscaled vertex weights); FM levels do not maintain it
  if (!pw_exact) {
    rc = K.weights(g0, K.loc(cur));
    if (rc) return rc;
  }
  // one host read for the cut and the part weights
  std::vector<int64_t> pw(k);
  unsigned long long cut2 = 0;
  HS_CHECK_CUDA(cudaMemcpyAsync(&cut2, cut_dev, 8, cudaMemcpyDeviceToHost, s));
  HS_CHECK_CUDA(cudaMemcpyAsync(pw.data(), K.d_pw, k * 8, cudaMemcpyDeviceToHost, s));
  int32_t ctl_h[16];
  HS_CHECK_CUDA(cudaMemcpyAsync(ctl_h, K.ctl, sizeof ctl_h, cudaMemcpyDeviceToHost, s));
  HS_CHECK_CUDA(cudaStreamSynchronize(s));
  cudaFreeAsync(cut_dev, s);
  int64_t cut = (int64_t)(cut2 / 2);
  if (cached_cut && w_uniform) cut *= w_uniform;
  rc = K.check_peers();
  if (rc) return rc;
  K.free_rep(cur);
  K.timer.mark("stats");
  double maxdev = 0;
  for (int p = 0; p < k; ++p)
    maxdev = std::max(maxdev, fabs((double)pw[p] / (double)K.total_vw - tpwgts_host[p]));
  const int64_t passes = ctl_h[CTL_PASSES];
  if (stats_host) {
    stats_host[0] = cut;
    stats_host[1] = (int64_t)K.levels.size();
    stats_host[2] = coarsest_n;
    stats_host[3] = (int64_t)llround(maxdev * 1e9);
    stats_host[4] = maxdev <= tol ? 1 : 0;
    stats_host[5] = passes;
    stats_host[6] = div;
    stats_host[7] = 0;
  }
  for (size_t i = 0; i < K.levels.size(); ++i) {
    Level &Lv = K.levels[i];
    if (Lv.cmap && !K.D.on()) cudaFreeAsync(Lv.cmap, s);  // sharded: lives in the arena
    cudaFreeAsync(Lv.g.deg, s);
    if (Lv.own_adj) cudaFreeAsync(Lv.g.adj, s);
    if (Lv.own_wgt) cudaFreeAsync(Lv.g.wgt, s);
    if (Lv.own_xbeg_vw) { cudaFreeAsync(Lv.g.xbeg, s); cudaFreeAsync(Lv.g.vw, s); }
  }
  cudaFreeAsync(K.d_hi, s); cudaFreeAsync(K.d_lo, s); cudaFreeAsync(K.d_target, s);
  cudaFreeAsync(K.d_pw, s); cudaFreeAsync(K.d_flows, s); cudaFreeAsync(K.d_prob, s);
  cudaFreeAsync(K.d_cum, s); cudaFreeAsync(K.counter, s);
  cudaFreeAsync(K.ctl, s); cudaFreeAsync(K.d_nnz, s);
  if (K.d_dpw) cudaFreeAsync(K.d_dpw, s);
  if (K.d_arbuf) cudaFreeAsync(K.d_arbuf, s);
  // no runtime error may leak to the caller's next CUDA call
  const cudaError_t e = cudaGetLastError();
  HS_REQUIRE(e == cudaSuccess, HS_ECUDA, "k-way: %s", cudaGetErrorString(e));
  return HS_OK;
}
}  // namespace

extern "C" int hs_partition_kway(const hs_ugraph_t *ug, int32_t k, const double *tpwgts_host,
                                 double tol, uint64_t seed, int32_t *part_out,
                                 int64_t *stats_host, void *stream) {
  HS_REQUIRE(ug && tpwgts_host && part_out, HS_EINVAL, "hs_partition_kway: null argument");
  HS_REQUIRE(k >= 1 && k <= kMaxParts, HS_ELIMIT, "k must be in 1..%d", kMaxParts);
  HS_REQUIRE(ug->n >= 1, HS_EINVAL, "empty graph");
  HS_REQUIRE(ug->vwgt_i, HS_EINVAL, "k-way path needs integer vertex weights");
  return partition_impl(ug, 0, ug->n, nullptr, k, tpwgts_host, tol, seed, part_out, stats_host,
                        (cudaStream_t)stream);
}

extern "C" int hs_partition_kway_starts(const hs_ugraph_t *ug, int32_t k,
                                        const double *tpwgts_host, double tol, uint64_t seed,
                                        const int32_t *starts, int32_t n_starts, int32_t *part_out,
                                        int64_t *stats_host, void *stream) {
  HS_REQUIRE(ug && tpwgts_host && part_out, HS_EINVAL, "hs_partition_kway_starts: null argument");
  HS_REQUIRE(k >= 1 && k <= kMaxParts, HS_ELIMIT, "k must be in 1..%d", kMaxParts);
  HS_REQUIRE(ug->n >= 1, HS_EINVAL, "empty graph");
  HS_REQUIRE(ug->vwgt_i, HS_EINVAL, "k-way path needs integer vertex weights");
  HS_REQUIRE(n_starts >= 0 && (n_starts == 0 || starts), HS_EINVAL, "starts missing");
  HS_REQUIRE(n_starts == 0 || ug->n <= kFmMaxLevel, HS_ELIMIT,
             "start partitions are taken for graphs of at most %d vertices", kFmMaxLevel);
  return partition_impl(ug, 0, ug->n, nullptr, k, tpwgts_host, tol, seed, part_out, stats_host,
                        (cudaStream_t)stream, starts, n_starts);
}

extern "C" int64_t hs_kway_dist_arena_bytes(int32_t n_global) {
  // parts of every level, one refinement state (4n), the fine->coarse maps
  // of every level (levels shrink geometrically: sum <= 24n with slack),
  // 256-byte rounding per array
  return (int64_t)kArenaHeader + 24ll * (int64_t)n_global + (1ll << 20);
}

extern "C" int hs_partition_kway_dist(const hs_ugraph_t *ug, int32_t v0, int32_t n_global,
                                      const hs_dist_t *dist, int32_t k,
                                      const double *tpwgts_host, double tol, uint64_t seed,
                                      int32_t *part_out, int64_t *stats_host, void *stream) {
  HS_REQUIRE(ug && dist && tpwgts_host && part_out, HS_EINVAL,
             "hs_partition_kway_dist: null argument");
  HS_REQUIRE(k >= 1 && k <= kMaxParts, HS_ELIMIT, "k must be in 1..%d", kMaxParts);
  HS_REQUIRE(dist->size >= 1 && dist->size <= kMaxRanks && dist->rank >= 0 &&
                 dist->rank < dist->size, HS_EINVAL, "bad group (rank %d of %d, max %d ranks)",
             dist->rank, dist->size, kMaxRanks);
  HS_REQUIRE(ug->n >= 1 && v0 >= 0 && (int64_t)v0 + ug->n <= n_global, HS_EINVAL,
             "rank range [%d, %lld) outside [0, %d) or empty", v0, (long long)v0 + ug->n,
             n_global);
  HS_REQUIRE(ug->vwgt_i, HS_EINVAL, "k-way path needs integer vertex weights");
  HS_REQUIRE(!ug->twin, HS_EINVAL, "sharded partition takes no twin index");
  if (dist->size == 1) {
    HS_REQUIRE(v0 == 0 && ug->n == n_global, HS_EINVAL, "a 1-rank group owns the whole graph");
    return partition_impl(ug, 0, n_global, nullptr, k, tpwgts_host, tol, seed, part_out,
                          stats_host, (cudaStream_t)stream);
  }
  for (int r = 0; r < dist->size; ++r)
    HS_REQUIRE(dist->arena[r], HS_EINVAL, "arena of rank %d missing", r);
  HS_REQUIRE(dist->arena_bytes >= hs_kway_dist_arena_bytes(n_global), HS_ELIMIT,
             "arena of %lld bytes < hs_kway_dist_arena_bytes(%d)", (long long)dist->arena_bytes,
             n_global);
  return partition_impl(ug, v0, n_global, dist, k, tpwgts_host, tol, seed, part_out, stats_host,
                        (cudaStream_t)stream);
}
