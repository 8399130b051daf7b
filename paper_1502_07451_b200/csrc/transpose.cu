// Device construction of a DAG's in-CSR from its out-CSR (the derived half of
// the TaskGraph container: `in_edges` in ascending-predecessor order,
// graph.py:89-90, next to the sorted out-lists of graph.py:73-81).
//
// A caller that holds only the sorted edge list (src, dst) — e.g. a host
// TaskGraph shipped to the GPU, or METIS-style input — copies the out-CSR and
// builds the rest here instead of moving a second copy of every edge over
// PCIe. Steps: (dst, src<<32|edge id) pairs, a stable LSD radix sort by
// destination over ceil(log2 n) bits (CUB onesweep), in_ptr from the run
// boundaries of the sorted keys, and a split of the values. Edges arrive
// sorted by (src, dst), so every destination's run keeps ascending sources:
// the reference order, bit-identical on every run. (An atomic-cursor scatter
// plus per-segment sorts measured 14 ms on config 4 — returning atomics and
// random 4-byte stores — against 3.5 ms here.)
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"

namespace {

// (src << 32 | edge id) of every edge, and a copy of its destination as the
// sort key. One warp per 32 consecutive sources: their out-lists are one
// contiguous range of out_dst, read coalesced; each edge's source comes from
// a 5-step search over the chunk's row pointers in shared memory.
constexpr int kWarps = 8;
__global__ void __launch_bounds__(kWarps * 32)
edge_pairs(int32_t n, const int64_t *__restrict__ out_ptr, const int32_t *__restrict__ out_dst,
           int32_t *key, uint64_t *val) {
  __shared__ int64_t s_ob[kWarps][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t nchunks = ((int64_t)n + 31) / 32;
  const int64_t wtot = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t c = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; c < nchunks; c += wtot) {
    const int64_t v0 = c * 32;
    const int cnt = (int)(n - v0 < 32 ? n - v0 : 32);
    if (lane < cnt) s_ob[w][lane] = out_ptr[v0 + lane];
    const int64_t e0 = out_ptr[v0], e1 = out_ptr[v0 + cnt];
    __syncwarp();
    for (int64_t e = e0 + lane; e < e1; e += 32) {
      int t = 0;
      for (int st = 16; st; st >>= 1)
        if (t + st < cnt && s_ob[w][t + st] <= e) t += st;
      key[e] = __ldg(out_dst + e);
      val[e] = ((uint64_t)(uint32_t)(v0 + t) << 32) | (uint32_t)e;
    }
    __syncwarp();
  }
}

// in_ptr from the destination-sorted keys: entry i starts every node d in
// (key[i-1], key[i]] (key[-1] = -1, key[m] = n).
__global__ void ptr_from_keys(int64_t m, int32_t n, const int32_t *__restrict__ key,
                              int64_t *in_ptr) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int prev = i == 0 ? -1 : __ldg(key + i - 1);
    const int cur = i == m ? n : __ldg(key + i);
    for (int d = prev + 1; d <= cur; ++d) in_ptr[d] = i;
  }
}

__global__ void split_pairs(int64_t m, const uint64_t *__restrict__ val, int32_t *src,
                            int32_t *eid) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t x = val[i];
    src[i] = (int32_t)(x >> 32);
    eid[i] = (int32_t)(uint32_t)x;
  }
}

struct Trace {  // HS_TRANSPOSE_TRACE=1: per-phase device times on stderr
  cudaStream_t s;
  bool on = getenv("HS_TRANSPOSE_TRACE") != nullptr;
  cudaEvent_t last = nullptr;
  explicit Trace(cudaStream_t st) : s(st) { mark(nullptr); }
  void mark(const char *name) {
    if (!on) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, s);
    if (name && last) {
      cudaEventSynchronize(e);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, last, e);
      fprintf(stderr, "[transpose] %-10s %8.3f ms\n", name, ms);
    }
    last = e;
  }
};

}  // namespace

static int transpose_radix(int32_t n, int64_t m, const int64_t *out_ptr, const int32_t *out_dst,
                    int64_t *in_ptr, int32_t *in_src, int32_t *in_eid, cudaStream_t s, Trace &tr) {
  // stable LSD radix sort of the edges by destination over the id bits:
  // edges arrive sorted by (src, dst), so each destination's run comes out
  // in ascending source (= ascending edge id) order
  int bits = 1;
  while (bits < 31 && (1ll << bits) < (int64_t)n) ++bits;
  hs::Scratch<int32_t> k0, k1;
  hs::Scratch<uint64_t> v0, v1;
  HS_CHECK_CUDA(k0.alloc(m, s));
  HS_CHECK_CUDA(k1.alloc(m, s));
  HS_CHECK_CUDA(v0.alloc(m, s));
  HS_CHECK_CUDA(v1.alloc(m, s));
  tr.mark("alloc");
  const int64_t chunks = ((int64_t)n + 31) / 32;
  const int grid = (int)std::max<int64_t>(
      1, std::min<int64_t>((int64_t)hs::sm_count() * 8, (chunks + kWarps - 1) / kWarps));
  edge_pairs<<<grid, kWarps * 32, 0, s>>>(n, out_ptr, out_dst, k0, v0);
  HS_CHECK_LAUNCH();
  tr.mark("pairs");
  cub::DoubleBuffer<int32_t> kb(k0.p, k1.p);
  cub::DoubleBuffer<uint64_t> vb(v0.p, v1.p);
  size_t tb = 0;
  HS_CHECK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, kb, vb, (int64_t)m, 0, bits, s));
  hs::Scratch<char> tmp;
  HS_CHECK_CUDA(tmp.alloc(tb, s));
  HS_CHECK_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, kb, vb, (int64_t)m, 0, bits, s));
  hs::count_launch(1);
  tr.mark("radix");
  ptr_from_keys<<<hs::grid_for(m + 1, 256, hs::sm_count() * 16), 256, 0, s>>>(m, n, kb.Current(),
                                                                             in_ptr);
  HS_CHECK_LAUNCH();
  split_pairs<<<hs::grid_for(m, 256, hs::sm_count() * 16), 256, 0, s>>>(m, vb.Current(),
                                                                         in_src, in_eid);
  HS_CHECK_LAUNCH();
  tr.mark("split");
  return HS_OK;
}

extern "C" int hs_dag_transpose(int32_t n, int64_t m, const int64_t *out_ptr,
                                const int32_t *out_dst, int64_t *in_ptr, int32_t *in_src,
                                int32_t *in_eid, void *stream) {
  HS_REQUIRE(n >= 0 && m >= 0, HS_EINVAL, "hs_dag_transpose: negative size");
  HS_REQUIRE(out_ptr && in_ptr && (m == 0 || (out_dst && in_src && in_eid)), HS_EINVAL,
             "hs_dag_transpose: null argument");
  HS_REQUIRE(m < (1ll << 31) - 1, HS_ELIMIT, "hs_dag_transpose: needs < 2^31 edges");
  cudaStream_t s = (cudaStream_t)stream;
  // algorithmic: out_ptr + out_dst read, in_ptr + in_src + in_eid written
  hs::Prof P("dag_transpose", s, 16.0 * n + 12.0 * m);
  Trace tr(s);
  if (m == 0) {
    HS_CHECK_CUDA(cudaMemsetAsync(in_ptr, 0, ((size_t)n + 1) * sizeof(int64_t), s));
    return HS_OK;
  }
  return transpose_radix(n, m, out_ptr, out_dst, in_ptr, in_src, in_eid, s, tr);
}
