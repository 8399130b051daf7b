// gp_build for a batch of DAGs on the device (policies.py:102-108: the
// workload ratio, then partition_heuristic, partition.py:258-295), the pin
// array of the gp policy as output — config 5's 4096 partitions without a
// host round trip per graph:
//
//   gp_prepare  per graph (thread): the kernel graph fm_refine builds
//               (partition.py:153-158: inter-kernel edges in sorted order,
//               each kernel's neighbours in edge order), kernel weights,
//               r_cpu = T_gpu / (T_gpu + T_cpu) from the fsum totals
//               (costs.py:239-253), error flags;
//   gp_orders   the start orders: the stable descending-weight order, then
//               the restart shuffles (host-drawn with the reference's
//               random.Random, identical for every graph of one size);
//   hs_fm2_batch (fm2.cu) refines every (graph, order);
//   gp_pick     the winner by (not feasible, cut, err, assignment) — the
//               reference's key — or the degenerate all-GPU / all-CPU split,
//               written as the per-node pin array (1 = GPU, root 0).
#include "common.cuh"

namespace {

__device__ __forceinline__ int32_t kp(int32_t x, int32_t root) {
  return root >= 0 && x > root ? x - 1 : x;
}

__global__ void gp_count(hs_dag_batch_t g, int64_t *n_kern, int64_t *n_edge) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= g.batch) return;
  const int64_t n0 = g.node_off[b], nb = g.node_off[b + 1] - n0;
  const int32_t root = g.root[b];
  const int64_t *op = g.out_ptr + n0 + b;
  const int32_t *od = g.out_dst + g.edge_off[b];
  int64_t ne = 0;
  for (int64_t u = 0; u < nb; ++u) {
    if (u == root) continue;
    for (int64_t e = op[u]; e < op[u + 1]; ++e) ne += od[e] != root;
  }
  n_kern[b] = nb - (root >= 0 ? 1 : 0);
  n_edge[b] = ne;
}

// flags[b]: 1 no kernels, 2 zero total kernel time, 4 zero kernel weight
__global__ void gp_prepare(hs_dag_batch_t g, const int64_t *koff, const int64_t *adj_off,
                           const int64_t *eoff, const double *tot, int64_t *xadj,
                           int32_t *adjncy, double *adjwgt, int32_t *eu, int32_t *ev, double *ew,
                           double *wk, double *r_cpu, int32_t *cursor, int32_t *flags) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= g.batch) return;
  const int64_t n0 = g.node_off[b], nb = g.node_off[b + 1] - n0, e0 = g.edge_off[b];
  const int32_t root = g.root[b];
  const int64_t *op = g.out_ptr + n0 + b;
  const int32_t *od = g.out_dst + e0;
  const int64_t k0 = koff[b], nk = koff[b + 1] - k0;
  int64_t *xa = xadj + k0 + b;  // nk + 1 local offsets
  int32_t *cur = cursor + k0;
  int flag = nk == 0 ? 1 : 0;
  const double tc = tot[3 * b], tg = tot[3 * b + 1];
  if (tc + tg == 0) flag |= 2;
  r_cpu[b] = flag & 2 ? 0.0 : tg / (tg + tc);
  bool any = false;
  for (int64_t x = 0; x < nb; ++x) {
    if (x == root) continue;
    const double w = g.w_gpu[n0 + x];
    wk[k0 + kp((int32_t)x, root)] = w;
    any |= w != 0.0;
  }
  if (!any) flag |= 4;
  flags[b] = flag;
  // edges in sorted (src, dst) order, root edges dropped; degrees
  for (int64_t x = 0; x <= nk; ++x) xa[x] = 0;
  int64_t p = 0;
  for (int64_t u = 0; u < nb; ++u) {
    if (u == root) continue;
    for (int64_t e = op[u]; e < op[u + 1]; ++e) {
      const int32_t v = od[e];
      if (v == root) continue;
      const int32_t a = kp((int32_t)u, root), c = kp(v, root);
      eu[eoff[b] + p] = a;
      ev[eoff[b] + p] = c;
      ew[eoff[b] + p] = g.w_xfer[e0 + e];
      xa[a + 1] += 1;
      xa[c + 1] += 1;
      ++p;
    }
  }
  for (int64_t x = 0; x < nk; ++x) {
    xa[x + 1] += xa[x];
    cur[x] = (int32_t)xa[x];
  }
  // each kernel's neighbours in edge order (lexsort by (kernel, edge position))
  const int64_t a0 = adj_off[b];
  for (int64_t q = 0; q < p; ++q) {
    const int32_t a = eu[eoff[b] + q], c = ev[eoff[b] + q];
    const double w = ew[eoff[b] + q];
    adjncy[a0 + cur[a]] = c;
    adjwgt[a0 + cur[a]++] = w;
    adjncy[a0 + cur[c]] = a;
    adjwgt[a0 + cur[c]++] = w;
  }
}

// orders [G][R][n]: row 0 stable descending weight, rows 1.. the shuffles
__global__ void gp_orders(int32_t G, const int64_t *koff, const double *wk, int32_t R,
                          const int32_t *shuffles, int32_t *orders) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= G) return;
  const int64_t k0 = koff[b], n = koff[b + 1] - k0;
  int32_t *row = orders + R * k0;
  for (int64_t i = 0; i < n; ++i) {  // stable insertion sort by -w
    const double key = wk[k0 + i];
    int64_t j = i - 1;
    while (j >= 0 && wk[k0 + row[j]] < key) {
      row[j + 1] = row[j];
      --j;
    }
    row[j + 1] = (int32_t)i;
  }
  for (int r = 1; r < R; ++r)
    for (int64_t i = 0; i < n; ++i) row[r * n + i] = shuffles[(r - 1) * n + i];
}

__global__ void gp_pick(hs_dag_batch_t g, const int64_t *koff, int32_t R, const double *r_cpu,
                        double tol, const int8_t *assign, const double *cut, const double *err,
                        int8_t *pin) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= g.batch) return;
  const int64_t k0 = koff[b], n = koff[b + 1] - k0, n0 = g.node_off[b];
  const int64_t nb = g.node_off[b + 1] - n0;
  const int32_t root = g.root[b];
  const double r = r_cpu[b];
  const int8_t *rows = assign + R * k0;
  int best = -1;
  if (!(r == 0.0 || r == 1.0)) {
    best = 0;
    for (int k = 1; k < R; ++k) {
      const bool fk = err[b * R + k] <= tol, fb = err[b * R + best] <= tol;
      bool better;
      if (fk != fb) better = fk;
      else if (cut[b * R + k] != cut[b * R + best]) better = cut[b * R + k] < cut[b * R + best];
      else if (err[b * R + k] != err[b * R + best]) better = err[b * R + k] < err[b * R + best];
      else {
        better = false;
        for (int64_t i = 0; i < n; ++i) {
          const int8_t x = rows[k * n + i], y = rows[best * n + i];
          if (x != y) {
            better = x < y;
            break;
          }
        }
      }
      if (better) best = k;
    }
  }
  for (int64_t x = 0; x < nb; ++x) {
    int8_t p = 0;
    if (x != root) {
      const int64_t i = kp((int32_t)x, root);
      p = best < 0 ? (r == 0.0 ? 1 : 0) : rows[best * n + i];
    }
    pin[n0 + x] = p;
  }
}

}  // namespace

extern "C" int hs_fm2_batch(int32_t G, const int64_t *node_off, const int64_t *adj_off,
                            const int64_t *edge_off, int64_t total_nodes, int32_t max_n,
                            const int64_t *xadj, const int32_t *adjncy, const double *adjwgt,
                            const double *edge_w, const int32_t *edge_u, const int32_t *edge_v,
                            const double *weights, const double *r_cpu, double tol,
                            const int32_t *orders, int32_t n_orders, int8_t *assign, double *cut,
                            double *err, int32_t *status, void *stream);
extern "C" int hs_exact_totals_batch(const hs_dag_batch_t *g, int include_root, double *out,
                                     void *stream);

extern "C" int hs_gp_pins_batch(const hs_dag_batch_t *g, int32_t restarts,
                                const int32_t *shuffles, int32_t n_shuffle, double tol,
                                int8_t *pin, int32_t *flags_host, void *stream) {
  HS_REQUIRE(g && pin && flags_host && restarts >= 0, HS_EINVAL,
             "hs_gp_pins_batch: bad argument");
  HS_REQUIRE(restarts == 0 || shuffles, HS_EINVAL, "hs_gp_pins_batch: shuffles missing");
  const int32_t G = g->batch;
  if (G == 0) return HS_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const int R = restarts + 1;
  hs::Scratch<int64_t> cnt;  // [2][G]: kernels, edges
  HS_CHECK_CUDA(cnt.alloc(2 * (int64_t)G, s));
  const int grid = (G + 63) / 64;
  gp_count<<<grid, 64, 0, s>>>(*g, cnt, cnt.p + G);
  HS_CHECK_LAUNCH();
  std::vector<int64_t> h(2 * (size_t)G);
  HS_CHECK_CUDA(cudaMemcpyAsync(h.data(), cnt, 2 * G * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  HS_CHECK_CUDA(cudaStreamSynchronize(s));
  std::vector<int64_t> koff(G + 1, 0), eoff(G + 1, 0), aoff(G + 1, 0);
  int64_t max_n = 0;
  for (int b = 0; b < G; ++b) {
    koff[b + 1] = koff[b] + h[b];
    eoff[b + 1] = eoff[b] + h[G + b];
    aoff[b + 1] = aoff[b] + 2 * h[G + b];
    max_n = h[b] > max_n ? h[b] : max_n;
    HS_REQUIRE(restarts == 0 || h[b] == n_shuffle, HS_EINVAL,
               "hs_gp_pins_batch: graph %d has %lld kernels, the shuffles %d", b,
               (long long)h[b], n_shuffle);
  }
  HS_REQUIRE(G <= 65535, HS_ELIMIT, "at most 65535 graphs per batch");
  const int64_t NK = koff[G], NE = eoff[G];
  hs::Scratch<int64_t> dkoff, deoff, daoff, xadj;
  hs::Scratch<int32_t> adjncy, eu, ev, cursor, flags, orders, status;
  hs::Scratch<double> adjwgt, ew, wk, r, tot, cut, err;
  hs::Scratch<int8_t> assign;
  HS_CHECK_CUDA(dkoff.alloc(G + 1, s));
  HS_CHECK_CUDA(deoff.alloc(G + 1, s));
  HS_CHECK_CUDA(daoff.alloc(G + 1, s));
  HS_CHECK_CUDA(xadj.alloc(NK + G, s));
  HS_CHECK_CUDA(adjncy.alloc(2 * NE, s));
  HS_CHECK_CUDA(adjwgt.alloc(2 * NE, s));
  HS_CHECK_CUDA(eu.alloc(NE, s));
  HS_CHECK_CUDA(ev.alloc(NE, s));
  HS_CHECK_CUDA(ew.alloc(NE, s));
  HS_CHECK_CUDA(wk.alloc(NK, s));
  HS_CHECK_CUDA(cursor.alloc(NK, s));
  HS_CHECK_CUDA(flags.alloc(G, s));
  HS_CHECK_CUDA(r.alloc(G, s));
  HS_CHECK_CUDA(tot.alloc(3 * (int64_t)G, s));
  HS_CHECK_CUDA(orders.alloc((int64_t)R * NK, s));
  HS_CHECK_CUDA(assign.alloc((int64_t)R * NK, s));
  HS_CHECK_CUDA(cut.alloc((int64_t)R * G, s));
  HS_CHECK_CUDA(err.alloc((int64_t)R * G, s));
  HS_CHECK_CUDA(status.alloc((int64_t)R * G, s));
  HS_CHECK_CUDA(cudaMemcpyAsync(dkoff, koff.data(), (G + 1) * 8, cudaMemcpyHostToDevice, s));
  HS_CHECK_CUDA(cudaMemcpyAsync(deoff, eoff.data(), (G + 1) * 8, cudaMemcpyHostToDevice, s));
  HS_CHECK_CUDA(cudaMemcpyAsync(daoff, aoff.data(), (G + 1) * 8, cudaMemcpyHostToDevice, s));
  HS_CHECK_CUDA(cudaMemsetAsync(status, 0, (int64_t)R * G * 4, s));
  int rc = hs_exact_totals_batch(g, 0, tot, stream);
  if (rc) return rc;
  gp_prepare<<<grid, 64, 0, s>>>(*g, dkoff, daoff, deoff, tot, xadj, adjncy, adjwgt, eu, ev, ew,
                                 wk, r, cursor, flags);
  HS_CHECK_LAUNCH();
  gp_orders<<<grid, 64, 0, s>>>(G, dkoff, wk, R, shuffles, orders);
  HS_CHECK_LAUNCH();
  HS_CHECK_CUDA(cudaMemcpyAsync(flags_host, flags, G * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  HS_CHECK_CUDA(cudaStreamSynchronize(s));
  for (int b = 0; b < G; ++b)
    if (flags_host[b]) return HS_OK;  // the caller raises the reference's error
  rc = hs_fm2_batch(G, dkoff, daoff, deoff, NK, (int32_t)max_n, xadj, adjncy, adjwgt, ew, eu, ev,
                    wk, r, tol, orders, R, assign, cut, err, status, stream);
  if (rc) return rc;
  gp_pick<<<grid, 64, 0, s>>>(*g, dkoff, R, r, tol, assign, cut, err, pin);
  HS_CHECK_LAUNCH();
  HS_CHECK_CUDA(cudaStreamSynchronize(s));  // scratch is released on return
  return HS_OK;
}
