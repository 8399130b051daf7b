// K0 exact totals and K2 evaluate (two-way and k-way) on the directed DAG CSR.
//
// Reference: partition.evaluate / _finish (pkg/src/hetsched/partition.py:60-84),
// graph.total_weights (graph.py:327-332), costs.workload_ratio
// (costs.py:239-253).
#include <cstdlib>

#include "common.cuh"
#include "numeric.cuh"

namespace {

using hs::kAccLimbs;

__device__ __forceinline__ int kpos(int v, int root) { return (root < 0 || v < root) ? v : v - 1; }

// ---------------------------------------------------------------- K0 -----
// acc layout: [3][kAccLimbs] int64 (w_cpu, w_gpu, w_xfer).
__global__ void totals_kernel(hs_dag_t g, int include_root, unsigned long long *acc) {
  __shared__ unsigned long long sacc[3 * kAccLimbs];
  for (int i = threadIdx.x; i < 3 * kAccLimbs; i += blockDim.x) sacc[i] = 0;
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < g.n; v += stride) {
    if (!include_root && v == g.root) continue;
    hs::superacc_split(g.w_cpu[v], [&](int li, int64_t c) {
      atomicAdd(&sacc[li], (unsigned long long)c);
    });
    hs::superacc_split(g.w_gpu[v], [&](int li, int64_t c) {
      atomicAdd(&sacc[kAccLimbs + li], (unsigned long long)c);
    });
  }
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < g.m; e += stride)
    hs::superacc_split(g.w_xfer[e], [&](int li, int64_t c) {
      atomicAdd(&sacc[2 * kAccLimbs + li], (unsigned long long)c);
    });
  __syncthreads();
  for (int i = threadIdx.x; i < 3 * kAccLimbs; i += blockDim.x)
    if (sacc[i]) atomicAdd(&acc[i], sacc[i]);
}

__global__ void round_kernel(const unsigned long long *acc, int count, double *out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < count) out[i] = hs::superacc_round((const int64_t *)(acc + (int64_t)i * kAccLimbs));
}

// ---------------------------------------------------------------- K2 -----
// mode 0: reference order, CPython sum() semantics (partition.py:62-69).
// The sums are order-dependent (Neumaier-compensated, not associative), so
// each stays one sequential chain: its cost is one dependent fp64 add per
// kept term. Everything else runs beside it: eval2_flags marks the cut
// edges of every assignment in parallel; eval2_seq gives each (sum,
// assignment) a 2-warp CTA where warp 0 streams the terms (coalesced,
// filtered and compacted in order into a shared-memory chunk) while lane 0 of
// warp 1 adds the previous chunk, double-buffered.
__global__ void eval2_flags(hs_dag_t g, const int8_t *part, uint8_t *flags) {
  const int b = blockIdx.y;
  const int nk = g.n - 1;
  const int8_t *p = part + (int64_t)b * nk;
  uint8_t *f = flags + (int64_t)b * g.m;
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < g.n;
       u += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e0 = g.out_ptr[u], e1 = g.out_ptr[u + 1];
    if (u == g.root) {
      for (int64_t e = e0; e < e1; ++e) f[e] = 0;
      continue;
    }
    const int8_t pu = p[kpos((int)u, g.root)];
    for (int64_t e = e0; e < e1; ++e) {
      const int v = g.out_dst[e];
      f[e] = (v != g.root && pu != p[kpos(v, g.root)]) ? 1 : 0;
    }
  }
}

constexpr int kSeqChunk = 1024;  // terms per producer step (32 per lane)

__global__ void __launch_bounds__(64) eval2_seq(hs_dag_t g, const int8_t *part,
                                                const uint8_t *flags, int src_gpu, double *cut,
                                                double *cpu_w, double *total) {
  __shared__ double buf[2][kSeqChunk];
  __shared__ int cnt[2];
  const int which = blockIdx.x, b = blockIdx.y;
  const int nk = g.n - 1;
  const int8_t *p = part + (int64_t)b * nk;
  const uint8_t *f = flags + (int64_t)b * g.m;
  const double *w = src_gpu ? g.w_gpu : g.w_cpu;
  const int64_t len = which == 0 ? g.m : (int64_t)g.n;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  hs::PySum acc;
  const int64_t steps = (len + kSeqChunk - 1) / kSeqChunk;
  for (int64_t it = 0; it <= steps; ++it) {
    if (warp == 0 && it < steps) {  // producer: terms [it*chunk, +chunk) -> buf[it & 1]
      double *out = buf[it & 1];
      int c = 0;
      const int64_t base = it * kSeqChunk;
      double val[32];
      bool keep[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int64_t i = base + j * 32 + lane;
        keep[j] = false;
        val[j] = 0.0;
        // unconditional loads: none waits for a flag, all 64 are in flight
        if (i < len) {
          if (which == 0) {
            keep[j] = __ldg(f + i) != 0;
            val[j] = __ldg(g.w_xfer + i);
          } else {
            const int v = (int)i;
            keep[j] = v != g.root && (which == 2 || __ldg(p + kpos(v, g.root)) == 0);
            val[j] = __ldg(w + v);
          }
        }
      }
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const unsigned m = __ballot_sync(0xffffffffu, keep[j]);
        if (keep[j]) out[c + __popc(m & ((1u << lane) - 1))] = val[j];
        c += __popc(m);
      }
      if (lane == 0) cnt[it & 1] = c;
    }
    if (warp == 1 && lane == 0 && it > 0) {  // consumer: the previous chunk, in order
      const double *in = buf[(it - 1) & 1];
      const int c = cnt[(it - 1) & 1];
      int i = 0;
      if (!acc.started && c > 0) acc.add(in[i++]);
      // PySum::add without the first-term branch; the terms are loaded 8
      // ahead so only the dependent adds are on the chain
      double f = acc.f, cc = acc.c;
      for (; i + 8 <= c; i += 8) {
        double x[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = in[i + j];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const double t = f + x[j];
          cc += fabs(f) >= fabs(x[j]) ? (f - t) + x[j] : (x[j] - t) + f;
          f = t;
        }
      }
      for (; i < c; ++i) {
        const double x = in[i];
        const double t = f + x;
        cc += fabs(f) >= fabs(x) ? (f - t) + x : (x - t) + f;
        f = t;
      }
      acc.f = f;
      acc.c = cc;
    }
    __syncthreads();
  }
  if (warp == 1 && lane == 0) {
    const double r = acc.started ? acc.result() : 0.0;
    if (which == 0) cut[b] = r;
    else if (which == 1) cpu_w[b] = r;
    else total[b] = r;
  }
}

// mode 1: correctly rounded sums, all nodes/edges in parallel.
// acc layout: [batch][3][kAccLimbs]; blockIdx.y = assignment.
__global__ void eval2_exact(hs_dag_t g, const int8_t *part, int src_gpu,
                            unsigned long long *acc) {
  __shared__ unsigned long long sacc[3 * kAccLimbs];
  for (int i = threadIdx.x; i < 3 * kAccLimbs; i += blockDim.x) sacc[i] = 0;
  __syncthreads();
  const int b = blockIdx.y;
  const int nk = g.n - 1;
  const int8_t *p = part + (int64_t)b * nk;
  const double *w = src_gpu ? g.w_gpu : g.w_cpu;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < g.n; u += stride) {
    if (u == g.root) continue;
    int8_t pu = p[kpos((int)u, g.root)];
    double wu = w[u];
    if (pu == 0)
      hs::superacc_split(wu, [&](int li, int64_t c) {
        atomicAdd(&sacc[kAccLimbs + li], (unsigned long long)c);
      });
    hs::superacc_split(wu, [&](int li, int64_t c) {
      atomicAdd(&sacc[2 * kAccLimbs + li], (unsigned long long)c);
    });
    for (int64_t e = g.out_ptr[u]; e < g.out_ptr[u + 1]; ++e) {
      int v = g.out_dst[e];
      if (v == g.root || p[kpos(v, g.root)] == pu) continue;
      hs::superacc_split(g.w_xfer[e], [&](int li, int64_t c) {
        atomicAdd(&sacc[li], (unsigned long long)c);
      });
    }
  }
  __syncthreads();
  unsigned long long *dst = acc + (int64_t)b * 3 * kAccLimbs;
  for (int i = threadIdx.x; i < 3 * kAccLimbs; i += blockDim.x)
    if (sacc[i]) atomicAdd(&dst[i], sacc[i]);
}

__global__ void eval2_exact_round(const unsigned long long *acc, int batch, double *cut,
                                  double *cpu_w, double *total) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= batch) return;
  const int64_t *a = (const int64_t *)(acc + (int64_t)b * 3 * kAccLimbs);
  cut[b] = hs::superacc_round(a);
  cpu_w[b] = hs::superacc_round(a + kAccLimbs);
  total[b] = hs::superacc_round(a + 2 * kAccLimbs);
}

// k-way evaluation. Integer sums are order-independent, so block partials +
// atomics stay deterministic.
constexpr int kMaxK = 64;

// Thread per source vertex (one assignment per blockIdx.y): the out-list is
// walked in ascending destination order, so the first edge into each foreign
// part pays the transfer; every lane is busy on task DAGs with ~10
// successors (a warp per vertex idled 2/3 of its lanes: 1.44 vs 0.72 ms).
__global__ void __launch_bounds__(256) evalk_thread(hs_dag_t g, const int32_t *part, int k,
                                                    const int64_t *vwgt, int64_t *cut_bytes,
                                                    int64_t *cut_edges, int64_t *loads,
                                                    int64_t *xcount, int64_t *xbytes,
                                                    int32_t *bad) {
  __shared__ unsigned long long s_load[kMaxK];
  __shared__ unsigned long long s_sum[4];
  const int b = blockIdx.y;
  const int32_t *p = part + (int64_t)b * g.n;
  for (int i = threadIdx.x; i < k; i += blockDim.x) s_load[i] = 0;
  if (threadIdx.x < 4) s_sum[threadIdx.x] = 0;
  __syncthreads();
  long long cb = 0, ce = 0, xc = 0, xb = 0;
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < g.n;
       u += (int64_t)gridDim.x * blockDim.x) {
    if (u == g.root) continue;
    const int pu = p[u];
    if ((unsigned)pu >= (unsigned)k) {  // no out-of-range shared/shift access
      atomicExch((int *)&bad[b], 1);
      continue;
    }
    atomicAdd(&s_load[pu], (unsigned long long)vwgt[u]);
    const int64_t e1 = g.out_ptr[u + 1];
    uint64_t seen = 0;  // parts already charged a transfer for u's item
    for (int64_t e = g.out_ptr[u]; e < e1; ++e) {
      const int v = __ldg(g.out_dst + e);
      if (v == g.root) continue;
      const int pv = __ldg(p + v);
      if (pv == pu) continue;
      if ((unsigned)pv >= (unsigned)k) {
        atomicExch((int *)&bad[b], 1);
        continue;
      }
      const int64_t by = __ldg(g.bytes + e);
      cb += by;
      ce += 1;
      if (!((seen >> pv) & 1ull)) {
        seen |= 1ull << pv;
        xc += 1;
        xb += by;
      }
    }
  }
  for (int off = 16; off; off >>= 1) {
    cb += __shfl_down_sync(0xffffffffu, cb, off);
    ce += __shfl_down_sync(0xffffffffu, ce, off);
    xc += __shfl_down_sync(0xffffffffu, xc, off);
    xb += __shfl_down_sync(0xffffffffu, xb, off);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&s_sum[0], (unsigned long long)cb);
    atomicAdd(&s_sum[1], (unsigned long long)ce);
    atomicAdd(&s_sum[2], (unsigned long long)xc);
    atomicAdd(&s_sum[3], (unsigned long long)xb);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    atomicAdd((unsigned long long *)&cut_bytes[b], s_sum[0]);
    atomicAdd((unsigned long long *)&cut_edges[b], s_sum[1]);
    atomicAdd((unsigned long long *)&xcount[b], s_sum[2]);
    atomicAdd((unsigned long long *)&xbytes[b], s_sum[3]);
  }
  for (int i = threadIdx.x; i < k; i += blockDim.x)
    if (s_load[i]) atomicAdd((unsigned long long *)&loads[(int64_t)b * k + i], s_load[i]);
}

// An assignment holding a part id outside [0, k) on a non-root node reports
// cut_edges = xfer_count = -1 (its other outputs are meaningless).
__global__ void evalk_flag(const int32_t *bad, int batch, int64_t *cut_edges, int64_t *xcount) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < batch && bad[b]) {
    cut_edges[b] = -1;
    xcount[b] = -1;
  }
}

}  // namespace

extern "C" int hs_exact_totals(const hs_dag_t *g, int include_root, double *out_host,
                               void *stream) {
  HS_REQUIRE(g && out_host, HS_EINVAL, "hs_exact_totals: null argument");
  cudaStream_t s = (cudaStream_t)stream;
  hs::Scratch<unsigned long long> acc;
  hs::Scratch<double> out;
  HS_CHECK_CUDA(acc.alloc(3 * kAccLimbs, s));
  HS_CHECK_CUDA(out.alloc(3, s));
  HS_CHECK_CUDA(cudaMemsetAsync(acc, 0, 3 * kAccLimbs * sizeof(unsigned long long), s));
  int64_t work = g->n > g->m ? g->n : g->m;
  totals_kernel<<<hs::grid_for(work, 256, hs::sm_count() * 4), 256, 0, s>>>(*g, include_root, acc);
  HS_CHECK_LAUNCH();
  round_kernel<<<1, 32, 0, s>>>(acc, 3, out);
  HS_CHECK_LAUNCH();
  HS_CHECK_CUDA(cudaMemcpyAsync(out_host, out, 3 * sizeof(double), cudaMemcpyDeviceToHost, s));
  HS_CHECK_CUDA(cudaStreamSynchronize(s));
  return HS_OK;
}

extern "C" int hs_evaluate2(const hs_dag_t *g, const int8_t *part, int32_t batch,
                            int weight_source, int mode, double *cut, double *cpu_w,
                            double *total, void *stream) {
  HS_REQUIRE(g && part && cut && cpu_w && total, HS_EINVAL, "hs_evaluate2: null argument");
  HS_REQUIRE(mode == 0 || mode == 1, HS_EINVAL, "hs_evaluate2: mode must be 0 or 1");
  if (batch <= 0) return HS_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (mode == 0) {
    hs::Scratch<uint8_t> flags;
    HS_CHECK_CUDA(flags.alloc((size_t)batch * (g->m > 0 ? g->m : 1), s));
    {
      hs::Prof P("evaluate2_flags", s, (double)batch * (8.0 * g->n + 5.0 * g->m + 1.0 * g->n +
                                                        1.0 * g->m));
      eval2_flags<<<dim3(hs::grid_for(g->n, 256, hs::sm_count() * 4), batch), 256, 0, s>>>(
          *g, part, flags);
    }
    HS_CHECK_LAUNCH();
    {
      hs::Prof P("evaluate2_ordered_sums", s, (double)batch * (9.0 * g->m + 17.0 * g->n));
      eval2_seq<<<dim3(3, batch), 64, 0, s>>>(*g, part, flags, weight_source, cut, cpu_w, total);
    }
    HS_CHECK_LAUNCH();
    return HS_OK;
  }
  hs::Scratch<unsigned long long> acc;
  size_t nacc = (size_t)batch * 3 * kAccLimbs;
  HS_CHECK_CUDA(acc.alloc(nacc, s));
  HS_CHECK_CUDA(cudaMemsetAsync(acc, 0, nacc * sizeof(unsigned long long), s));
  dim3 grid(hs::grid_for(g->n, 256, hs::sm_count() * 4), batch);
  eval2_exact<<<grid, 256, 0, s>>>(*g, part, weight_source, acc);
  HS_CHECK_LAUNCH();
  eval2_exact_round<<<(batch + 63) / 64, 64, 0, s>>>(acc, batch, cut, cpu_w, total);
  HS_CHECK_LAUNCH();
  return HS_OK;
}

extern "C" int hs_evaluate_kway(const hs_dag_t *g, const int32_t *part, int32_t batch,
                                int32_t k, const int64_t *vwgt_i, int64_t *cut_bytes,
                                int64_t *cut_edges, int64_t *loads, int64_t *xfer_count,
                                int64_t *xfer_bytes, void *stream) {
  HS_REQUIRE(g && part && vwgt_i && cut_bytes && cut_edges && loads && xfer_count && xfer_bytes,
             HS_EINVAL, "hs_evaluate_kway: null argument");
  HS_REQUIRE(k >= 1 && k <= kMaxK, HS_ELIMIT, "k must be in 1..%d", kMaxK);
  if (batch <= 0) return HS_OK;
  cudaStream_t s = (cudaStream_t)stream;
  HS_CHECK_CUDA(cudaMemsetAsync(cut_bytes, 0, batch * sizeof(int64_t), s));
  HS_CHECK_CUDA(cudaMemsetAsync(cut_edges, 0, batch * sizeof(int64_t), s));
  HS_CHECK_CUDA(cudaMemsetAsync(xfer_count, 0, batch * sizeof(int64_t), s));
  HS_CHECK_CUDA(cudaMemsetAsync(xfer_bytes, 0, batch * sizeof(int64_t), s));
  HS_CHECK_CUDA(cudaMemsetAsync(loads, 0, (size_t)batch * k * sizeof(int64_t), s));
  hs::Scratch<int32_t> bad;
  HS_CHECK_CUDA(bad.alloc(batch, s));
  HS_CHECK_CUDA(cudaMemsetAsync(bad, 0, batch * sizeof(int32_t), s));
  {
    // per assignment: out_ptr, out_dst, bytes, part[dst] gather, part[src], vwgt
    hs::Prof P("evaluate_kway", s, (double)batch * (8.0 * (g->n + 1) + 4.0 * g->m + 8.0 * g->m +
                                                    4.0 * g->m + 4.0 * g->n + 8.0 * g->n));
    dim3 tgrid(hs::grid_for((int64_t)g->n, 256, hs::sm_count() * 8), batch);
    evalk_thread<<<tgrid, 256, 0, s>>>(*g, part, k, vwgt_i, cut_bytes, cut_edges, loads,
                                       xfer_count, xfer_bytes, bad);
  }
  HS_CHECK_LAUNCH();
  evalk_flag<<<(batch + 255) / 256, 256, 0, s>>>(bad, batch, cut_edges, xfer_count);
  HS_CHECK_LAUNCH();
  return HS_OK;
}

namespace {
// one block per graph of a batch: exact (fsum) totals of w_cpu, w_gpu over the
// graph's non-root nodes (include_root = 0) and of w_xfer over its edges
__global__ void totals_batch_kernel(hs_dag_batch_t g, int include_root, double *out) {
  __shared__ unsigned long long sacc[3 * kAccLimbs];
  for (int i = threadIdx.x; i < 3 * kAccLimbs; i += blockDim.x) sacc[i] = 0;
  __syncthreads();
  const int b = blockIdx.x;
  const int64_t n0 = g.node_off[b], n1 = g.node_off[b + 1];
  const int64_t e0 = g.edge_off[b], e1 = g.edge_off[b + 1];
  const int root = g.root[b];
  for (int64_t v = n0 + threadIdx.x; v < n1; v += blockDim.x) {
    if (!include_root && v - n0 == root) continue;
    hs::superacc_split(g.w_cpu[v], [&](int li, int64_t c) {
      atomicAdd(&sacc[li], (unsigned long long)c);
    });
    hs::superacc_split(g.w_gpu[v], [&](int li, int64_t c) {
      atomicAdd(&sacc[kAccLimbs + li], (unsigned long long)c);
    });
  }
  for (int64_t e = e0 + threadIdx.x; e < e1; e += blockDim.x)
    hs::superacc_split(g.w_xfer[e], [&](int li, int64_t c) {
      atomicAdd(&sacc[2 * kAccLimbs + li], (unsigned long long)c);
    });
  __syncthreads();
  if (threadIdx.x < 3)
    out[3 * b + threadIdx.x] = hs::superacc_round((const int64_t *)(sacc + threadIdx.x * kAccLimbs));
}
}  // namespace

extern "C" int hs_exact_totals_batch(const hs_dag_batch_t *g, int include_root, double *out,
                                     void *stream) {
  HS_REQUIRE(g && out, HS_EINVAL, "hs_exact_totals_batch: null argument");
  if (g->batch == 0) return HS_OK;
  totals_batch_kernel<<<g->batch, 128, 0, (cudaStream_t)stream>>>(*g, include_root, out);
  HS_CHECK_LAUNCH();
  return HS_OK;
}
