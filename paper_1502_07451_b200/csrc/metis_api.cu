// METIS-compatible entry point over the k-way partitioner.
//
// The paper hands its task DAG to METIS and the
// reference exports METIS files (graphio.py:277-304). A caller of
// METIS_PartGraphKway (idx_t = int32, real_t = float, host arrays) can link
// hs_METIS_PartGraphKway instead: same arguments, same outputs (part, objval),
// computed by hs_partition_kway on the current device.
#include "common.cuh"
#include <vector>
#include <algorithm>

extern "C" int hs_METIS_PartGraphKway(const int32_t *nvtxs, const int32_t *ncon,
                                      const int32_t *xadj, const int32_t *adjncy,
                                      const int32_t *vwgt, const int32_t *vsize,
                                      const int32_t *adjwgt, const int32_t *nparts,
                                      const float *tpwgts, const float *ubvec,
                                      const int32_t *options, int32_t *objval, int32_t *part) {
  (void)vsize;
  (void)options;
  HS_REQUIRE(nvtxs && xadj && adjncy && nparts && part, HS_EINVAL, "METIS API: null argument");
  HS_REQUIRE(!ncon || *ncon == 1, HS_ELIMIT, "only ncon = 1 is supported");
  const int n = *nvtxs, k = *nparts;
  HS_REQUIRE(n >= 1 && k >= 1, HS_EINVAL, "METIS API: empty graph or no parts");
  const int64_t nnz = xadj[n];
  // METIS semantics: max part weight <= ubvec * target; here |w_p/W - t_p| <= tol
  std::vector<double> tp(k);
  for (int p = 0; p < k; ++p) tp[p] = tpwgts ? (double)tpwgts[p] : 1.0 / k;
  const double ub = ubvec ? (double)ubvec[0] : 1.03;
  const double tol = (ub - 1.0) * *std::min_element(tp.begin(), tp.end());
  cudaStream_t s = 0;
  std::vector<int64_t> hx(n + 1);
  for (int i = 0; i <= n; ++i) hx[i] = xadj[i];
  std::vector<int32_t> hv(n, 1), hw(std::max<int64_t>(nnz, 1), 1);
  if (vwgt) std::copy(vwgt, vwgt + n, hv.begin());
  if (adjwgt) std::copy(adjwgt, adjwgt + nnz, hw.begin());
  hs::Scratch<int64_t> dx;
  hs::Scratch<int32_t> da, dw, dv, dp;
  HS_CHECK_CUDA(dx.alloc(n + 1, s));
  HS_CHECK_CUDA(da.alloc(nnz, s));
  HS_CHECK_CUDA(dw.alloc(nnz, s));
  HS_CHECK_CUDA(dv.alloc(n, s));
  HS_CHECK_CUDA(dp.alloc(n, s));
  HS_CHECK_CUDA(cudaMemcpyAsync(dx, hx.data(), (n + 1) * 8, cudaMemcpyHostToDevice, s));
  if (nnz) {
    HS_CHECK_CUDA(cudaMemcpyAsync(da, adjncy, nnz * 4, cudaMemcpyHostToDevice, s));
    HS_CHECK_CUDA(cudaMemcpyAsync(dw, hw.data(), nnz * 4, cudaMemcpyHostToDevice, s));
  }
  HS_CHECK_CUDA(cudaMemcpyAsync(dv, hv.data(), n * 4, cudaMemcpyHostToDevice, s));
  hs_ugraph_t g;
  g.n = n;
  g.nnz = nnz;
  g.xadj = dx;
  g.adjncy = da;
  g.adjwgt = nullptr;
  g.adjwgt_i = dw;
  g.vwgt = nullptr;
  g.vwgt_i = dv;
  g.twin = nullptr;
  int64_t stats[8] = {0};
  int rc = hs_partition_kway(&g, k, tp.data(), tol, 0, dp, stats, s);
  if (rc) return rc;
  HS_CHECK_CUDA(cudaMemcpyAsync(part, dp, n * 4, cudaMemcpyDeviceToHost, s));
  HS_CHECK_CUDA(cudaStreamSynchronize(s));
  if (objval) *objval = (int32_t)std::min<int64_t>(stats[0], INT32_MAX);
  return HS_OK;
}
