// Device weight attachment (attach_weights, graph.py:308-324) for CSR graphs:
// per node the two kernel times of its (kind, size), per edge the transfer
// time of its byte count (costs.py:44-55, 82-139).
//
// The host hands over one entry per distinct (kind, size) pair the graph
// uses: a closed form the device evaluates per node (the synthetic model's
// MA: c * size^2 [+ launch], MM: c * size^3 [+ launch], costs.py:87-100 —
// size^2 and size^3 are exact below 2^26 and rounded once above, as
// CPython's float ** int on an integer-valued float), a value pair the host
// read from the model once (calibration tables, custom models), zero (SOURCE
// kind, and the root) or "no cost entry" (the first such node, in the
// caller's node order, is reported). Transfers are latency + bytes /
// bandwidth in IEEE fp64 (the reference's float expression; no FMA in this
// file: the library is built with --fmad=false), or a per-edge value.
#include "common.cuh"

namespace {

enum : int32_t { kFormTable = 0, kFormMA = 1, kFormMM = 2, kFormZero = 3, kFormError = -1 };

__global__ void node_weights(hs_cost_table_t t, int32_t n, const int32_t *pair,
                             const int64_t *size, const int32_t *rank, double *w_cpu,
                             double *w_gpu, int32_t *bad_rank) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int32_t p = pair[v];
    const int32_t form = (p >= 0 && p < t.n_pairs) ? t.form[p] : kFormError;
    double c = 0.0, g = 0.0;
    if (form == kFormTable) {
      c = t.cpu[p];
      g = t.gpu[p];
    } else if (form == kFormMA || form == kFormMM) {
      const double x = (double)size[v];
      const double work = form == kFormMA ? x * x : (x * x) * x;
      c = (form == kFormMA ? t.ma_cpu : t.mm_cpu) * work;
      g = (form == kFormMA ? t.ma_gpu : t.mm_gpu) * work + t.launch_ms;
    } else if (form == kFormError) {
      atomicMin(bad_rank, rank ? rank[v] : (int32_t)v);
    }
    w_cpu[v] = c;
    w_gpu[v] = g;
  }
}

__global__ void edge_weights(hs_cost_table_t t, int64_t m, const int64_t *bytes,
                             const double *xfer_tab, double *w_xfer, unsigned long long *bad) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x) {
    if (xfer_tab) {
      w_xfer[e] = xfer_tab[e];
      continue;
    }
    const int64_t b = bytes[e];
    if (b < 0) {
      atomicMin(bad, (unsigned long long)e);
      w_xfer[e] = 0.0;
      continue;
    }
    w_xfer[e] = t.latency_ms + (double)b / t.bandwidth;
  }
}

}  // namespace

extern "C" int hs_attach_weights(const hs_cost_table_t *t, int32_t n, const int32_t *pair,
                                 const int64_t *size, const int32_t *rank, double *w_cpu,
                                 double *w_gpu, int64_t m, const int64_t *bytes,
                                 const double *xfer_tab, double *w_xfer, int32_t *bad_node_host,
                                 int64_t *bad_edge_host, void *stream) {
  HS_REQUIRE(t && bad_node_host && bad_edge_host, HS_EINVAL, "hs_attach_weights: null argument");
  HS_REQUIRE(n >= 0 && m >= 0, HS_EINVAL, "hs_attach_weights: negative size");
  HS_REQUIRE(n == 0 || (pair && size && w_cpu && w_gpu), HS_EINVAL,
             "hs_attach_weights: null node array");
  HS_REQUIRE(m == 0 || (w_xfer && (bytes || xfer_tab)), HS_EINVAL,
             "hs_attach_weights: null edge array");
  HS_REQUIRE(xfer_tab || m == 0 || t->bandwidth > 0.0, HS_EINVAL,
             "hs_attach_weights: bandwidth must be > 0");
  cudaStream_t s = (cudaStream_t)stream;
  hs::Scratch<int32_t> bad_rank;
  hs::Scratch<unsigned long long> bad_edge;
  HS_CHECK_CUDA(bad_rank.alloc(1, s));
  HS_CHECK_CUDA(bad_edge.alloc(1, s));
  static const int32_t kNone = 0x7fffffff;  // static: the async copy reads it later
  HS_CHECK_CUDA(cudaMemcpyAsync(bad_rank, &kNone, sizeof kNone, cudaMemcpyHostToDevice, s));
  HS_CHECK_CUDA(cudaMemsetAsync(bad_edge, 0xff, sizeof(unsigned long long), s));
  if (n > 0) {
    node_weights<<<hs::grid_for(n, 256), 256, 0, s>>>(*t, n, pair, size, rank, w_cpu, w_gpu,
                                                      bad_rank);
    HS_CHECK_LAUNCH();
  }
  if (m > 0) {
    edge_weights<<<hs::grid_for(m, 256), 256, 0, s>>>(*t, m, bytes, xfer_tab, w_xfer, bad_edge);
    HS_CHECK_LAUNCH();
  }
  int32_t r = 0;
  unsigned long long e = 0;
  HS_CHECK_CUDA(cudaMemcpyAsync(&r, bad_rank, sizeof r, cudaMemcpyDeviceToHost, s));
  HS_CHECK_CUDA(cudaMemcpyAsync(&e, bad_edge, sizeof e, cudaMemcpyDeviceToHost, s));
  HS_CHECK_CUDA(cudaStreamSynchronize(s));
  *bad_node_host = r == kNone ? -1 : r;
  *bad_edge_host = e == ~0ull ? -1 : (int64_t)e;
  return HS_OK;
}
