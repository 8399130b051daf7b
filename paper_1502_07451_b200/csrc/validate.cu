// Device validation of a task-DAG CSR — the checks of the reference's
// validate (pkg/src/hetsched/graph.py:113-150) that a CSR can violate:
//   node loop (graph.py:125-129): negative weights, non-zero weights on the
//     root (the SOURCE node, graph.py:128);
//   edge loop (graph.py:130-140): self-loops, negative transfer weights,
//     negative byte counts;
//   topological_order (graph.py:153-172): Kahn with self-loops ignored in
//     the in-degrees; on a cycle, the smallest id never released;
//   initial kernels (graph.py:145-148): non-root nodes without predecessors.
// Duplicate ids/edges, unknown endpoints and the root's kind only exist in
// the object model and stay on the host (graph.py:116-124).
//
// Kahn's released set does not depend on the pop order, so a level-
// synchronous release (cooperative kernel, grid barrier per level) finds the
// same stuck nodes as the reference's min-heap.
#include "common.cuh"

namespace {

enum : int8_t { kNegWeight = 1, kRootWeight = 2, kNoPred = 4, kStuck = 8 };
enum : int8_t { kSelfLoop = 1, kNegXfer = 2, kNegBytes = 4 };

struct VArgs {
  hs_dag_t g;
  int8_t *node_bad, *edge_bad;
  unsigned long long *count;  // [7]
  int32_t *first;             // [7]
  int32_t *indeg, *front[2], *fcount;  // Kahn state
  unsigned *bar;              // [2]
};

struct Barrier {
  unsigned *count, *gen;
  __device__ void sync(unsigned nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned g0 = *(volatile unsigned *)gen;
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

__device__ __forceinline__ void note(VArgs &A, int check, int32_t idx) {
  atomicAdd(&A.count[check], 1ull);
  atomicMin(&A.first[check], idx);
}

__global__ void validate_kernel(VArgs A) {
  const hs_dag_t &g = A.g;
  Barrier bar{A.bar, A.bar + 1};
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  // node and edge checks; Kahn in-degrees without self-loops
  for (int64_t v = tid; v < g.n; v += stride) {
    int8_t bad = 0;
    if (g.w_cpu[v] < 0 || g.w_gpu[v] < 0) { bad |= kNegWeight; note(A, 0, (int32_t)v); }
    if (v == g.root && (g.w_cpu[v] != 0 || g.w_gpu[v] != 0)) { bad |= kRootWeight; note(A, 1, (int32_t)v); }
    const int64_t i0 = g.in_ptr[v], i1 = g.in_ptr[v + 1];
    if (v != g.root && i1 == i0) { bad |= kNoPred; note(A, 6, (int32_t)v); }
    int32_t d = 0;
    for (int64_t j = i0; j < i1; ++j) d += g.in_src[j] != (int32_t)v;
    A.indeg[v] = d;
    if (d == 0) A.front[0][atomicAdd(&A.fcount[0], 1)] = (int32_t)v;
    for (int64_t e = g.out_ptr[v]; e < g.out_ptr[v + 1]; ++e) {
      int8_t eb = 0;
      if (g.out_dst[e] == (int32_t)v) { eb |= kSelfLoop; note(A, 2, (int32_t)e); }
      if (g.w_xfer[e] < 0) { eb |= kNegXfer; note(A, 3, (int32_t)e); }
      if (g.bytes[e] < 0) { eb |= kNegBytes; note(A, 4, (int32_t)e); }
      if (A.edge_bad) A.edge_bad[e] = eb;
    }
    if (A.node_bad) A.node_bad[v] = bad;
  }
  bar.sync(gridDim.x);
  // level-synchronous Kahn: release every node whose in-degree reaches 0
  for (int it = 0;; ++it) {
    const int cur = it & 1, nxt = cur ^ 1;
    const int32_t ncur = __ldcg(&A.fcount[cur]);
    if (ncur == 0) break;
    for (int64_t i = tid; i < ncur; i += stride) {
      const int v = __ldcg(&A.front[cur][i]);
      for (int64_t e = g.out_ptr[v]; e < g.out_ptr[v + 1]; ++e) {
        const int s = g.out_dst[e];
        if (s != v && atomicSub(&A.indeg[s], 1) == 1)
          A.front[nxt][atomicAdd(&A.fcount[nxt], 1)] = s;
      }
    }
    bar.sync(gridDim.x);
    if (tid == 0) A.fcount[cur] = 0;
    bar.sync(gridDim.x);
  }
  // never released: on or after a cycle
  for (int64_t v = tid; v < g.n; v += stride)
    if (__ldcg(&A.indeg[v]) > 0) {
      note(A, 5, (int32_t)v);
      if (A.node_bad) A.node_bad[v] |= kStuck;
    }
}

}  // namespace

extern "C" int hs_validate_dag(const hs_dag_t *g, int64_t *counts_host, int32_t *first_host,
                               int8_t *node_bad, int8_t *edge_bad, void *stream) {
  HS_REQUIRE(g && counts_host && first_host, HS_EINVAL, "hs_validate_dag: null argument");
  HS_REQUIRE(g->n >= 1 && g->root >= 0 && g->root < g->n, HS_EINVAL,
             "hs_validate_dag: root %d outside [0, %d)", g->root, g->n);
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t n = g->n;
  hs::Scratch<int32_t> st;
  hs::Scratch<unsigned long long> cnt;
  HS_CHECK_CUDA(st.alloc(3 * n + 16, s));
  HS_CHECK_CUDA(cnt.alloc(7, s));
  VArgs A;
  A.g = *g;
  A.node_bad = node_bad;
  A.edge_bad = edge_bad;
  A.count = cnt;
  A.indeg = st.p;
  A.front[0] = st.p + n;
  A.front[1] = st.p + 2 * n;
  A.first = st.p + 3 * n;                 // [7]
  A.fcount = st.p + 3 * n + 8;            // [2]
  A.bar = (unsigned *)(st.p + 3 * n + 10);  // [2]
  HS_CHECK_CUDA(cudaMemsetAsync(cnt, 0, 7 * sizeof(unsigned long long), s));
  HS_CHECK_CUDA(cudaMemsetAsync(A.first, 0x7f, 7 * sizeof(int32_t), s));
  HS_CHECK_CUDA(cudaMemsetAsync(A.fcount, 0, 4 * sizeof(int32_t), s));
  const int block = 256;
  int per_sm = 0;
  HS_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, validate_kernel, block, 0));
  int grid = hs::sm_count() * (per_sm < 4 ? per_sm : 4);
  const int need = (int)((n + block - 1) / block);
  if (grid > need) grid = need;
  if (grid < 1) grid = 1;
  void *args[] = {&A};
  HS_CHECK_CUDA(cudaLaunchCooperativeKernel((void *)validate_kernel, grid, block, args, 0, s));
  HS_CHECK_LAUNCH();
  int32_t first[7];
  HS_CHECK_CUDA(cudaMemcpyAsync(counts_host, cnt, 7 * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  HS_CHECK_CUDA(cudaMemcpyAsync(first, A.first, sizeof first, cudaMemcpyDeviceToHost, s));
  HS_CHECK_CUDA(cudaStreamSynchronize(s));
  for (int i = 0; i < 7; ++i) first_host[i] = counts_host[i] ? first[i] : -1;
  return HS_OK;
}
