// K5/K6 (exact two-way) — the reference partitioner on the device.
//
// One CTA per start order runs, with the reference's exact arithmetic:
//   _greedy_init    partition.py:223-236  (sequential over the order)
//   _repair_balance partition.py:239-255  (parallel argmin per flip)
//   fm_refine       partition.py:137-220  (parallel argmax per move)
// and reports the refined assignment with the cut/err _finish would store
// (partition.py:76-84). The host picks the winner by the reference key
// (not feasible, cut, err, lex) (partition.py:291-294).
//
// Exactness: every `sum(...)` of the reference is a PySum in the reference's
// iteration order (numeric.cuh); `+=` loops are plain sequential adds; gains
// are recomputed from scratch in adjacency order whenever a neighbour moves
// (a node's gain only depends on its neighbours' sides), never updated
// incrementally; ties break toward the smaller kernel position exactly as
// the reference's ascending scans with strict comparisons do.
#include "common.cuh"
#include "numeric.cuh"

namespace {

constexpr int kThreads = 512;

struct FmArgs {
  int n;
  const int64_t *xadj;
  const int32_t *adjncy;
  const double *adjwgt;
  const double *ew;       // inter-kernel edges, sorted order
  const int32_t *eu, *ev;
  int64_t ne;
  const double *w;
  double r, tol;
  const int32_t *orders;  // [R][n] or null
  const int8_t *start;    // [n] or null
  int8_t *assign;         // [R][n] out (the `assignment`)
  double *cut_out, *err_out;
  int32_t *status;        // [R]
  // scratch [R][n]
  int8_t *work;
  int8_t *locked;
  double *gain;
  int32_t *trail;
};

struct Best {
  double key;  // gain (argmax) or new_err (argmin)
  int idx;
  double aux;  // new_cpu
};

// Block-wide arg-reduction. maximize: larger key wins; else smaller wins;
// equal keys -> smaller idx. idx < 0 means "no candidate".
__device__ Best block_reduce(Best b, bool maximize, Best *sbuf) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  auto better = [&](const Best &x, const Best &y) {  // x beats y?
    if (x.idx < 0) return false;
    if (y.idx < 0) return true;
    if (x.key != y.key) return maximize ? x.key > y.key : x.key < y.key;
    return x.idx < y.idx;
  };
  for (int off = 16; off; off >>= 1) {
    Best o;
    o.key = __shfl_down_sync(0xffffffffu, b.key, off);
    o.idx = __shfl_down_sync(0xffffffffu, b.idx, off);
    o.aux = __shfl_down_sync(0xffffffffu, b.aux, off);
    if (better(o, b)) b = o;
  }
  if (lane == 0) sbuf[wid] = b;
  __syncthreads();
  if (wid == 0) {
    const int nw = blockDim.x >> 5;
    b = lane < nw ? sbuf[lane] : Best{0.0, -1, 0.0};
    for (int off = 16; off; off >>= 1) {
      Best o;
      o.key = __shfl_down_sync(0xffffffffu, b.key, off);
      o.idx = __shfl_down_sync(0xffffffffu, b.idx, off);
      o.aux = __shfl_down_sync(0xffffffffu, b.aux, off);
      if (better(o, b)) b = o;
    }
    if (lane == 0) sbuf[0] = b;
  }
  __syncthreads();
  Best r = sbuf[0];
  __syncthreads();
  return r;
}

// err_of / the evaluate() balance error: cpu_w = PySum over CPU kernels in id order.
__device__ double cpu_weight(const int8_t *a, const double *w, int n) {
  hs::PySum s;
  for (int i = 0; i < n; ++i)
    if (a[i] == 0) s.add(w[i]);
  return s.started ? s.result() : 0.0;
}

// cut_of: PySum of w_xfer over cut inter-kernel edges in sorted order.
__device__ double cut_of(const int8_t *a, const FmArgs &A) {
  hs::PySum s;
  for (int64_t e = 0; e < A.ne; ++e)
    if (a[A.eu[e]] != a[A.ev[e]]) s.add(A.ew[e]);
  return s.started ? s.result() : 0.0;
}

__device__ __forceinline__ double node_gain(int i, const int8_t *work, const FmArgs &A) {
  double g = 0.0;
  const int8_t si = work[i];
  for (int64_t j = A.xadj[i]; j < A.xadj[i + 1]; ++j) {
    double wj = A.adjwgt[j];
    g = g + (work[A.adjncy[j]] != si ? wj : -wj);
  }
  return g;
}

// key(cut, err) = (err > tol, cut) compared lexicographically
__device__ __forceinline__ bool key_less(bool ia, double ca, bool ib, double cb) {
  if (ia != ib) return !ia;
  return ca < cb;
}

__device__ void fm2_body(const FmArgs &A, const int o) {
  __shared__ Best sbuf[32];
  __shared__ double s_total, s_cpu, s_err, s_cut;
  __shared__ int s_flag;
  const int n = A.n;
  int8_t *asg = A.assign + (int64_t)o * n;
  int8_t *work = A.work + (int64_t)o * n;
  int8_t *locked = A.locked + (int64_t)o * n;
  double *gain = A.gain + (int64_t)o * n;
  int32_t *trail = A.trail + (int64_t)o * n;
  const double r = A.r, tol = A.tol;
  const int tid = threadIdx.x, T = blockDim.x;

  if (tid == 0) {
    hs::PySum t;
    for (int i = 0; i < n; ++i) t.add(A.w[i]);
    s_total = t.started ? t.result() : 0.0;
  }
  __syncthreads();
  const double total = s_total;
  if (total == 0.0) {
    if (tid == 0) A.status[o] = HS_EPARTITION;
    return;
  }

  if (A.start) {
    for (int i = tid; i < n; i += T) asg[i] = A.start[i];
    __syncthreads();
  } else {
    // _greedy_init: strictly-better test, sequential over the order
    if (tid == 0) {
      const int32_t *ord = A.orders + (int64_t)o * n;
      double cpu = 0.0;
      for (int k = 0; k < n; ++k) {
        int i = ord[k];
        double with_i = fabs((cpu + A.w[i]) / total - r);
        double without = fabs(cpu / total - r);
        if (with_i < without) { asg[i] = 0; cpu = cpu + A.w[i]; }
        else asg[i] = 1;
      }
      s_cpu = cpu_weight(asg, A.w, n);
      s_err = fabs(s_cpu / total - r);
    }
    __syncthreads();
    // _repair_balance: flip the first node with minimal new_err < err
    while (s_err > tol) {
      const double cpu = s_cpu, err = s_err;
      Best b{0.0, -1, 0.0};
      for (int i = tid; i < n; i += T) {
        double nc = cpu + (asg[i] == 1 ? A.w[i] : -A.w[i]);
        double ne = fabs(nc / total - r);
        if (ne < err && (b.idx < 0 || ne < b.key)) b = Best{ne, i, nc};
      }
      b = block_reduce(b, false, sbuf);
      if (b.idx < 0) break;
      if (tid == 0) {
        asg[b.idx] = asg[b.idx] == 1 ? 0 : 1;
        s_err = b.key;
        s_cpu = b.aux;
      }
      __syncthreads();
    }
  }

  // ---- fm_refine ----
  __syncthreads();  // every warp has read s_err in the loop test above
  if (tid == 0) {
    s_cut = cut_of(asg, A);
    s_err = fabs(cpu_weight(asg, A.w, n) / total - r);
  }
  __syncthreads();
  double best_cut = s_cut, best_err = s_err;
  bool improved = true;
  while (improved) {
    improved = false;
    for (int i = tid; i < n; i += T) { work[i] = asg[i]; locked[i] = 0; }
    __syncthreads();
    for (int i = tid; i < n; i += T) gain[i] = node_gain(i, work, A);
    if (tid == 0) {
      s_cpu = cpu_weight(work, A.w, n);
      s_err = fabs(s_cpu / total - r);  // err_of(work)
      s_cut = best_cut;
    }
    __syncthreads();
    double cur_cut = best_cut;
    double cur_err = s_err;
    double cpu = s_cpu;
    bool pk_inf = cur_err > tol;
    double pk_cut = cur_cut;
    int best_prefix = 0, ntrail = 0;
    while (ntrail < n) {
      Best b{0.0, -1, 0.0};
      for (int i = tid; i < n; i += T) {
        if (locked[i]) continue;
        double nc = cpu + (work[i] == 1 ? A.w[i] : -A.w[i]);
        double ne = fabs(nc / total - r);
        if (ne > tol && ne >= cur_err) continue;
        double g = gain[i];
        if (b.idx < 0 || g > b.key) b = Best{g, i, nc};
      }
      b = block_reduce(b, true, sbuf);
      if (b.idx < 0) break;
      const int x = b.idx;
      // every thread applies the (uniform) move to its registers
      cpu = b.aux;
      cur_err = fabs(cpu / total - r);
      cur_cut = cur_cut - b.key;
      if (tid == 0) {
        work[x] = work[x] == 1 ? 0 : 1;
        locked[x] = 1;
        trail[ntrail] = x;
      }
      ++ntrail;
      bool kinf = cur_err > tol;
      if (key_less(kinf, cur_cut, pk_inf, pk_cut)) {
        pk_inf = kinf; pk_cut = cur_cut; best_prefix = ntrail;
      }
      __syncthreads();
      // refresh the gains touched by the move: x and its neighbours
      const int64_t j0 = A.xadj[x], j1 = A.xadj[x + 1];
      for (int64_t j = j0 + tid; j < j1; j += T) {
        int y = A.adjncy[j];
        gain[y] = node_gain(y, work, A);
      }
      if (tid == 0) gain[x] = node_gain(x, work, A);
      __syncthreads();
    }
    if (best_prefix > 0) {
      if (tid == 0) {
        for (int t = 0; t < best_prefix; ++t) {
          int i = trail[t];
          asg[i] = asg[i] == 1 ? 0 : 1;
        }
        double nc = cut_of(asg, A);
        double ne = fabs(cpu_weight(asg, A.w, n) / total - r);
        if (key_less(ne > tol, nc, best_err > tol, best_cut)) {
          s_cut = nc; s_err = ne; s_flag = 1;
        } else {
          for (int t = 0; t < best_prefix; ++t) {
            int i = trail[t];
            asg[i] = asg[i] == 1 ? 0 : 1;
          }
          s_flag = 0;
        }
      }
      __syncthreads();
      if (s_flag) { best_cut = s_cut; best_err = s_err; improved = true; }
      __syncthreads();
    }
  }
  // _finish: evaluate() on the final assignment
  if (tid == 0) {
    A.cut_out[o] = cut_of(asg, A);
    A.err_out[o] = fabs(cpu_weight(asg, A.w, n) / total - r);
    A.status[o] = 0;
  }
}

__global__ void __launch_bounds__(kThreads) fm2_kernel(FmArgs A) { fm2_body(A, blockIdx.x); }

// Batched: blockIdx.y = graph, blockIdx.x = start order. Per-graph arrays are
// concatenated; xadj holds n_g + 1 local offsets per graph.
struct FmBatch {
  FmArgs base;
  const int64_t *node_off, *adj_off, *edge_off;
  const double *r;
  int R;
};

__global__ void __launch_bounds__(kThreads) fm2_batch_kernel(FmBatch Bt) {
  const int g = blockIdx.y;
  FmArgs A = Bt.base;
  const int64_t n0 = Bt.node_off[g];
  const int n = (int)(Bt.node_off[g + 1] - n0);
  const int64_t a0 = Bt.adj_off[g], e0 = Bt.edge_off[g];
  A.n = n;
  A.xadj = Bt.base.xadj + n0 + g;
  A.adjncy = Bt.base.adjncy + a0;
  A.adjwgt = Bt.base.adjwgt + a0;
  A.ew = Bt.base.ew + e0;
  A.eu = Bt.base.eu + e0;
  A.ev = Bt.base.ev + e0;
  A.ne = Bt.edge_off[g + 1] - e0;
  A.w = Bt.base.w + n0;
  A.r = Bt.r[g];
  const int64_t so = (int64_t)Bt.R * n0;
  A.orders = Bt.base.orders + so;
  A.assign = Bt.base.assign + so;
  A.work = Bt.base.work + so;
  A.locked = Bt.base.locked + so;
  A.gain = Bt.base.gain + so;
  A.trail = Bt.base.trail + so;
  A.cut_out = Bt.base.cut_out + (int64_t)g * Bt.R;
  A.err_out = Bt.base.err_out + (int64_t)g * Bt.R;
  A.status = Bt.base.status + (int64_t)g * Bt.R;
  if (n > 0) fm2_body(A, blockIdx.x);
}

// ---- brute_force_partition (partition.py:87-134) ----
// Mask bit (n-1-k) set = kernel k on GPU; ascending mask = lexicographic
// order, so "first minimum" = smallest mask among equal keys.
struct BfBest {
  double err; int64_t emask;
  double cut; int64_t cmask;
};

__global__ void brute2_kernel(int n, const double *w, double r, double tol,
                              const int32_t *ea, const int32_t *eb, const double *ewt,
                              int64_t ne, BfBest *partial) {
  __shared__ double s_total;
  __shared__ BfBest sb[32];
  if (threadIdx.x == 0) {
    hs::PySum t;
    for (int k = 0; k < n; ++k) t.add(w[k]);
    s_total = t.result();
  }
  __syncthreads();
  const double total = s_total;
  BfBest b{0.0, -1, 0.0, -1};
  const int64_t nmask = 1ll << n;
  for (int64_t mask = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; mask < nmask;
       mask += (int64_t)gridDim.x * blockDim.x) {
    double cpu = 0.0;
    for (int k = 0; k < n; ++k)
      if (!((mask >> (n - 1 - k)) & 1)) cpu = cpu + w[k];
    double err = fabs(cpu / total - r);
    if (b.emask < 0 || err < b.err || (err == b.err && mask < b.emask)) { b.err = err; b.emask = mask; }
    if (err <= tol) {
      double cut = 0.0;
      for (int64_t e = 0; e < ne; ++e)
        if (((mask >> (n - 1 - ea[e])) & 1) != ((mask >> (n - 1 - eb[e])) & 1)) cut = cut + ewt[e];
      if (b.cmask < 0 || cut < b.cut || (cut == b.cut && mask < b.cmask)) { b.cut = cut; b.cmask = mask; }
    }
  }
  // warp then block reduce
  auto merge = [](BfBest &x, const BfBest &y) {
    if (y.emask >= 0 && (x.emask < 0 || y.err < x.err || (y.err == x.err && y.emask < x.emask))) {
      x.err = y.err; x.emask = y.emask;
    }
    if (y.cmask >= 0 && (x.cmask < 0 || y.cut < x.cut || (y.cut == x.cut && y.cmask < x.cmask))) {
      x.cut = y.cut; x.cmask = y.cmask;
    }
  };
  for (int off = 16; off; off >>= 1) {
    BfBest o;
    o.err = __shfl_down_sync(0xffffffffu, b.err, off);
    o.emask = __shfl_down_sync(0xffffffffu, b.emask, off);
    o.cut = __shfl_down_sync(0xffffffffu, b.cut, off);
    o.cmask = __shfl_down_sync(0xffffffffu, b.cmask, off);
    merge(b, o);
  }
  if ((threadIdx.x & 31) == 0) sb[threadIdx.x >> 5] = b;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < (int)(blockDim.x >> 5); ++i) merge(b, sb[i]);
    partial[blockIdx.x] = b;
  }
}

__global__ void brute2_final(const BfBest *partial, int nb, const double *w, int n,
                             int64_t *out) {
  hs::PySum t;
  for (int k = 0; k < n; ++k) t.add(w[k]);
  out[2] = t.result() == 0.0;
  BfBest b = partial[0];
  for (int i = 1; i < nb; ++i) {
    const BfBest &y = partial[i];
    if (y.emask >= 0 && (b.emask < 0 || y.err < b.err || (y.err == b.err && y.emask < b.emask))) {
      b.err = y.err; b.emask = y.emask;
    }
    if (y.cmask >= 0 && (b.cmask < 0 || y.cut < b.cut || (y.cut == b.cut && y.cmask < b.cmask))) {
      b.cut = y.cut; b.cmask = y.cmask;
    }
  }
  out[0] = b.cmask >= 0 ? b.cmask : b.emask;
  out[1] = b.cmask >= 0 ? 1 : 0;
}

}  // namespace

extern "C" int hs_fm2(const hs_ugraph_t *g, const double *edge_w_sorted, const int32_t *edge_u,
                      const int32_t *edge_v, int64_t n_edges, const double *weights,
                      double r_cpu, double tol, const int32_t *orders, int32_t n_orders,
                      const int8_t *start, int8_t *assign, double *cut, double *err,
                      void *stream) {
  HS_REQUIRE(g && weights && assign && cut && err, HS_EINVAL, "hs_fm2: null argument");
  HS_REQUIRE(orders || start, HS_EINVAL, "hs_fm2: need orders or a start assignment");
  HS_REQUIRE(g->n > 0 && n_orders > 0, HS_EINVAL, "hs_fm2: empty problem");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t n = g->n, R = n_orders;
  hs::Scratch<int8_t> work, locked;
  hs::Scratch<double> gain;
  hs::Scratch<int32_t> trail, status;
  HS_CHECK_CUDA(work.alloc(R * n, s));
  HS_CHECK_CUDA(locked.alloc(R * n, s));
  HS_CHECK_CUDA(gain.alloc(R * n, s));
  HS_CHECK_CUDA(trail.alloc(R * n, s));
  HS_CHECK_CUDA(status.alloc(R, s));
  FmArgs A;
  A.n = (int)n;
  A.xadj = g->xadj; A.adjncy = g->adjncy; A.adjwgt = g->adjwgt;
  A.ew = edge_w_sorted; A.eu = edge_u; A.ev = edge_v; A.ne = n_edges;
  A.w = weights; A.r = r_cpu; A.tol = tol;
  A.orders = orders; A.start = start;
  A.assign = assign; A.cut_out = cut; A.err_out = err; A.status = status;
  A.work = work; A.locked = locked; A.gain = gain; A.trail = trail;
  int threads = n >= 4096 ? kThreads : (n >= 512 ? 256 : 128);
  fm2_kernel<<<(int)R, threads, 0, s>>>(A);
  HS_CHECK_LAUNCH();
  int32_t st[64];
  int32_t *hst = R <= 64 ? st : (int32_t *)malloc(R * sizeof(int32_t));
  HS_CHECK_CUDA(cudaMemcpyAsync(hst, status, R * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  HS_CHECK_CUDA(cudaStreamSynchronize(s));
  int bad = 0;
  for (int64_t i = 0; i < R; ++i)
    if (hst[i]) bad = hst[i];
  if (hst != st) free(hst);
  HS_REQUIRE(bad == 0, HS_EPARTITION, "zero total node weight; attach weights first");
  return HS_OK;
}

extern "C" int hs_brute2(int32_t n, const double *weights, double r_cpu, double tol,
                         const int32_t *edge_a, const int32_t *edge_b, const double *edge_w,
                         int64_t n_edges, int64_t *mask_host, int32_t *feasible_host,
                         void *stream) {
  HS_REQUIRE(n >= 1 && n <= 30, HS_ELIMIT, "brute force supports 1..30 kernels, got %d", n);
  HS_REQUIRE(weights && mask_host && feasible_host, HS_EINVAL, "hs_brute2: null argument");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t nmask = 1ll << n;
  const int block = 256;
  int grid = hs::grid_for(nmask, block, hs::sm_count() * 8);
  hs::Scratch<BfBest> partial;
  hs::Scratch<int64_t> out;
  HS_CHECK_CUDA(partial.alloc(grid, s));
  HS_CHECK_CUDA(out.alloc(3, s));
  brute2_kernel<<<grid, block, 0, s>>>(n, weights, r_cpu, tol, edge_a, edge_b, edge_w, n_edges,
                                       partial);
  HS_CHECK_LAUNCH();
  brute2_final<<<1, 1, 0, s>>>(partial, grid, weights, n, out);
  HS_CHECK_LAUNCH();
  int64_t h[3];
  HS_CHECK_CUDA(cudaMemcpyAsync(h, out, sizeof h, cudaMemcpyDeviceToHost, s));
  HS_CHECK_CUDA(cudaStreamSynchronize(s));
  HS_REQUIRE(!h[2], HS_EPARTITION, "zero total node weight; attach weights first");
  *mask_host = h[0];
  *feasible_host = (int32_t)h[1];
  return HS_OK;
}

extern "C" int hs_fm2_batch(int32_t G, const int64_t *node_off, const int64_t *adj_off,
                            const int64_t *edge_off, int64_t total_nodes, int32_t max_n,
                            const int64_t *xadj, const int32_t *adjncy, const double *adjwgt,
                            const double *edge_w, const int32_t *edge_u, const int32_t *edge_v,
                            const double *weights, const double *r_cpu, double tol,
                            const int32_t *orders, int32_t n_orders, int8_t *assign, double *cut,
                            double *err, int32_t *status, void *stream) {
  HS_REQUIRE(G >= 0 && n_orders > 0, HS_EINVAL, "hs_fm2_batch: bad sizes");
  if (G == 0) return HS_OK;
  HS_REQUIRE(G <= 65535, HS_ELIMIT, "at most 65535 graphs per batch");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t cells = (int64_t)n_orders * total_nodes;
  hs::Scratch<int8_t> work, locked;
  hs::Scratch<double> gain;
  hs::Scratch<int32_t> trail;
  HS_CHECK_CUDA(work.alloc(cells, s));
  HS_CHECK_CUDA(locked.alloc(cells, s));
  HS_CHECK_CUDA(gain.alloc(cells, s));
  HS_CHECK_CUDA(trail.alloc(cells, s));
  FmBatch Bt;
  memset(&Bt, 0, sizeof Bt);
  Bt.base.xadj = xadj; Bt.base.adjncy = adjncy; Bt.base.adjwgt = adjwgt;
  Bt.base.ew = edge_w; Bt.base.eu = edge_u; Bt.base.ev = edge_v;
  Bt.base.w = weights; Bt.base.tol = tol; Bt.base.orders = orders; Bt.base.start = nullptr;
  Bt.base.assign = assign; Bt.base.cut_out = cut; Bt.base.err_out = err; Bt.base.status = status;
  Bt.base.work = work; Bt.base.locked = locked; Bt.base.gain = gain; Bt.base.trail = trail;
  Bt.node_off = node_off; Bt.adj_off = adj_off; Bt.edge_off = edge_off; Bt.r = r_cpu;
  Bt.R = n_orders;
  const int threads = max_n >= 4096 ? kThreads : (max_n >= 512 ? 256 : (max_n >= 64 ? 64 : 32));
  {
    hs::Prof P("fm2_batch", s, 0.0);
    fm2_batch_kernel<<<dim3(n_orders, G), threads, 0, s>>>(Bt);
  }
  HS_CHECK_LAUNCH();
  return HS_OK;
}
