// Device generator of the layered fan-in task DAGs of configs 2 and 4.
//
// Family (generalising the reference's layered two-input
// generator graph.py:180-305 to fan-in ~m/n): n kernels (ids 1..n, root 0)
// over L = ceil(sqrt(n)) layers sized like graph.py:175-177; every kernel
// past layer 0 draws f(v) distinct predecessors uniformly from all kernels of
// earlier layers, f(v) = base + (rank(v) < rem) with m = base*K + rem spread
// over the K such kernels in id order (clamped to the kernels available);
// the root feeds every layer-0 kernel (graph.py:299-301). Draw j (attempt a)
// of kernel v is splitmix64(seed, v, a) mod avail, duplicates rejected.
// oracle/layered_oracle.py restates this bit for bit.
#include "common.cuh"
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

namespace {

struct Layout {
  int64_t n, L, q, r;
  __host__ __device__ explicit Layout(int64_t n_) : n(n_) {
    int64_t s = 0;
    while (s * s < n) ++s;  // ceil(sqrt(n)) exactly (host: loop is O(sqrt n))
    L = s < 1 ? 1 : s;
    if (L > n) L = n;
    q = n / L;
    r = n % L;
  }
  __host__ __device__ int64_t first(int64_t l) const {  // first kernel id of layer l
    return 1 + l * q + (l < r ? l : r);
  }
  __host__ __device__ int64_t layer(int64_t v) const {  // v: kernel id >= 1
    int64_t idx = v - 1, big = r * (q + 1);
    return idx < big ? idx / (q + 1) : r + (idx - big) / q;
  }
};

__host__ __device__ inline uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

__host__ __device__ inline int64_t fanin(const Layout &Lo, int64_t v, int64_t m) {
  int64_t l = Lo.layer(v);
  if (l == 0) return 1;  // the root edge
  int64_t size0 = Lo.first(1) - 1;
  int64_t K = Lo.n - size0;
  int64_t base = m / K, rem = m % K;
  int64_t rank = v - 1 - size0;
  int64_t f = base + (rank < rem ? 1 : 0);
  int64_t avail = Lo.first(l) - 1;
  return f < avail ? f : avail;
}

__global__ void degree_kernel(Layout Lo, int64_t m, int64_t *indeg) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v <= Lo.n;
       v += (int64_t)gridDim.x * blockDim.x)
    indeg[v] = v == 0 ? 0 : fanin(Lo, v, m);
}

constexpr int kMaxFanin = 64;

__global__ void draw_kernel(Layout Lo, int64_t m, uint64_t seed, const int64_t *in_ptr,
                            int32_t *in_src, int32_t *layer_of) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v <= Lo.n;
       v += (int64_t)gridDim.x * blockDim.x) {
    if (v == 0) { if (layer_of) layer_of[0] = -1; continue; }
    int64_t l = Lo.layer(v);
    if (layer_of) layer_of[v] = (int32_t)l;
    int32_t *dst = in_src + in_ptr[v];
    if (l == 0) { dst[0] = 0; continue; }
    int64_t f = in_ptr[v + 1] - in_ptr[v];
    int64_t avail = Lo.first(l) - 1;
    int32_t got[kMaxFanin];
    int nf = 0;
    uint64_t key = seed * 0x2545F4914F6CDD1Dull ^ ((uint64_t)v * 0x9E3779B97F4A7C15ull);
    for (uint64_t a = 0; nf < f; ++a) {
      int32_t u = (int32_t)(1 + splitmix64(key + a) % (uint64_t)avail);
      bool dup = false;
      for (int i = 0; i < nf; ++i) dup |= got[i] == u;
      if (!dup) {  // insertion keeps the row ascending
        int i = nf++;
        while (i > 0 && got[i - 1] > u) { got[i] = got[i - 1]; --i; }
        got[i] = u;
      }
    }
    for (int i = 0; i < nf; ++i) dst[i] = got[i];
  }
}

// key = (src << 24 | dst) in in-order; value = in position
__global__ void edge_keys(int64_t n, const int64_t *in_ptr, const int32_t *in_src,
                          uint64_t *keys, int32_t *vals) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v <= n;
       v += (int64_t)gridDim.x * blockDim.x)
    for (int64_t j = in_ptr[v]; j < in_ptr[v + 1]; ++j) {
      keys[j] = ((uint64_t)in_src[j] << 32) | (uint64_t)v;
      vals[j] = (int32_t)j;
    }
}

__global__ void out_fill(int64_t n_nodes, int64_t m, const uint64_t *keys, const int32_t *vals,
                         int64_t *out_ptr, int32_t *out_dst, int32_t *in_eid) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e <= m;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t s = e < m ? (int64_t)(keys[e] >> 32) : n_nodes;
    int64_t sp = e > 0 ? (int64_t)(keys[e - 1] >> 32) : -1;
    for (int64_t u = sp + 1; u <= s && u <= n_nodes; ++u) out_ptr[u] = e;
    if (e < m) {
      out_dst[e] = (int32_t)(keys[e] & 0xffffffffull);
      in_eid[vals[e]] = (int32_t)e;
    }
  }
}

}  // namespace

extern "C" int hs_layered_sizes(int64_t n_kernels, int64_t m_inter, int64_t *n_nodes_host,
                                int64_t *n_edges_host) {
  HS_REQUIRE(n_kernels >= 2 && n_kernels < (1ll << 31) - 1, HS_ELIMIT,
             "n_kernels must be in [2, 2^31-2]");
  HS_REQUIRE(m_inter >= 0, HS_EINVAL, "negative edge count");
  Layout Lo(n_kernels);
  HS_REQUIRE(Lo.L >= 2, HS_EINVAL, "need at least two layers");
  int64_t size0 = Lo.first(1) - 1;
  int64_t K = n_kernels - size0;
  HS_REQUIRE(m_inter / K < kMaxFanin, HS_ELIMIT, "mean fan-in must be < %d", kMaxFanin);
  int64_t base = m_inter / K, rem = m_inter % K, total = 0;
  for (int64_t l = 1; l < Lo.L; ++l) {
    int64_t lo = Lo.first(l), hi = Lo.first(l + 1), avail = lo - 1;
    // ranks [lo-1-size0, hi-1-size0); the first `rem` ranks get base+1
    int64_t r0 = lo - 1 - size0, r1 = hi - 1 - size0;
    int64_t plus = (rem > r0 ? (rem < r1 ? rem : r1) - r0 : 0);
    int64_t cnt = hi - lo;
    int64_t fp = base + 1 < avail ? base + 1 : avail, fb = base < avail ? base : avail;
    total += plus * fp + (cnt - plus) * fb;
  }
  *n_nodes_host = n_kernels + 1;
  *n_edges_host = total + size0;
  return HS_OK;
}

extern "C" int hs_layered_generate(int64_t n_kernels, int64_t m_inter, uint64_t seed,
                                   int64_t *out_ptr, int32_t *out_dst, int64_t *in_ptr,
                                   int32_t *in_src, int32_t *in_eid, int32_t *layer_of,
                                   void *stream) {
  int64_t n_nodes = 0, m = 0;
  int rc = hs_layered_sizes(n_kernels, m_inter, &n_nodes, &m);
  if (rc) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  Layout Lo(n_kernels);
  hs::Scratch<int64_t> indeg;
  HS_CHECK_CUDA(indeg.alloc(n_nodes + 1, s));
  int grid = hs::grid_for(n_nodes, 256);
  degree_kernel<<<grid, 256, 0, s>>>(Lo, m_inter, indeg);
  HS_CHECK_LAUNCH();
  HS_CHECK_CUDA(cudaMemsetAsync(indeg.p + n_nodes, 0, sizeof(int64_t), s));
  size_t tb = 0;
  HS_CHECK_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, indeg.p, in_ptr, n_nodes + 1, s));
  {
    hs::Scratch<char> tmp;
    HS_CHECK_CUDA(tmp.alloc(tb, s));
    HS_CHECK_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, indeg.p, in_ptr, n_nodes + 1, s));
  }
  draw_kernel<<<grid, 256, 0, s>>>(Lo, m_inter, seed, in_ptr, in_src, layer_of);
  HS_CHECK_LAUNCH();
  hs::Scratch<uint64_t> keys, keys2;
  hs::Scratch<int32_t> vals, vals2;
  HS_CHECK_CUDA(keys.alloc(m, s));
  HS_CHECK_CUDA(keys2.alloc(m, s));
  HS_CHECK_CUDA(vals.alloc(m, s));
  HS_CHECK_CUDA(vals2.alloc(m, s));
  edge_keys<<<grid, 256, 0, s>>>(n_kernels, in_ptr, in_src, keys, vals);
  HS_CHECK_LAUNCH();
  int bits = 1;
  while ((1ll << bits) <= n_nodes) ++bits;
  tb = 0;
  HS_CHECK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys.p, keys2.p, vals.p, vals2.p,
                                                m, 0, 32 + bits, s));
  {
    hs::Scratch<char> tmp;
    HS_CHECK_CUDA(tmp.alloc(tb, s));
    HS_CHECK_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, keys.p, keys2.p, vals.p, vals2.p,
                                                  m, 0, 32 + bits, s));
  }
  out_fill<<<hs::grid_for(m + 1, 256), 256, 0, s>>>(n_nodes, m, keys2, vals2, out_ptr, out_dst,
                                                    in_eid);
  HS_CHECK_LAUNCH();
  hs::count_launch(6);
  return HS_OK;
}
