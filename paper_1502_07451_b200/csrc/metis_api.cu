// METIS-compatible entry point over the k-way partitioner.
//
// The paper hands its task DAG to METIS and the
// reference exports METIS files (graphio.py:277-304). A caller of
// METIS_PartGraphKway (idx_t = int32, real_t = float, host arrays) links this
// library instead: same symbol, same arguments, same return convention
// (METIS_OK = 1, METIS_ERROR_INPUT = -2, METIS_ERROR_MEMORY = -3,
// METIS_ERROR = -4), same outputs (part, objval), computed by
// hs_partition_kway on the current device. hs_METIS_PartGraphKway is the
// same function under the library's prefix.
//
// Honoured options (METIS 5 option indices, -1 = default):
//   options[8]  METIS_OPTION_SEED       seed of the partitioner
//   options[16] METIS_OPTION_UFACTOR    imbalance x1000 when ubvec is NULL
//   options[17] METIS_OPTION_NUMBERING  0 = C (default), 1 = Fortran (1-based)
// Everything else (ptype, ctype, iptype, niter, ncuts, contig, ...) selects
// among METIS's own algorithms and has no counterpart here.
#include "common.cuh"
#include <vector>
#include <algorithm>

namespace {
constexpr int kMetisOk = 1, kMetisErrorInput = -2, kMetisErrorMemory = -3, kMetisError = -4;
constexpr int kOptSeed = 8, kOptUfactor = 16, kOptNumbering = 17;

int metis_status(int hs_rc) {
  if (hs_rc == HS_OK) return kMetisOk;
  if (hs_rc == HS_EINVAL || hs_rc == HS_ELIMIT || hs_rc == HS_EPARTITION) return kMetisErrorInput;
  return kMetisError;
}

int part_graph_kway(const int32_t *nvtxs, const int32_t *ncon, const int32_t *xadj,
                    const int32_t *adjncy, const int32_t *vwgt, const int32_t *adjwgt,
                    const int32_t *nparts, const float *tpwgts, const float *ubvec,
                    const int32_t *options, int32_t *objval, int32_t *part) {
  HS_REQUIRE(nvtxs && xadj && adjncy && nparts && part, HS_EINVAL, "METIS API: null argument");
  HS_REQUIRE(!ncon || *ncon == 1, HS_ELIMIT, "only ncon = 1 is supported");
  const int n = *nvtxs, k = *nparts;
  HS_REQUIRE(n >= 1 && k >= 1, HS_EINVAL, "METIS API: empty graph or no parts");
  auto opt = [&](int i) { return options ? options[i] : -1; };
  const int base = opt(kOptNumbering) == 1 ? 1 : 0;
  HS_REQUIRE(opt(kOptNumbering) <= 1, HS_EINVAL, "METIS API: numbering must be 0 or 1");
  HS_REQUIRE(xadj[0] == base, HS_EINVAL, "METIS API: xadj[0] must equal the numbering base");
  const int64_t nnz = (int64_t)xadj[n] - base;
  HS_REQUIRE(nnz >= 0, HS_EINVAL, "METIS API: xadj[n] < xadj[0]");
  // METIS semantics: max part weight <= ubvec * target; here |w_p/W - t_p| <= tol
  std::vector<double> tp(k);
  double tsum = 0.0;
  for (int p = 0; p < k; ++p) {
    tp[p] = tpwgts ? (double)tpwgts[p] : 1.0 / k;
    HS_REQUIRE(tp[p] >= 0.0, HS_EINVAL, "METIS API: negative tpwgts[%d]", p);
    tsum += tp[p];
  }
  HS_REQUIRE(tsum > 0.0, HS_EINVAL, "METIS API: tpwgts sum to zero");
  for (double &t : tp) t /= tsum;
  double ub = 1.03;  // METIS's default ufactor for k-way is 30
  if (ubvec) ub = (double)ubvec[0];
  else if (opt(kOptUfactor) >= 0) ub = 1.0 + opt(kOptUfactor) / 1000.0;
  HS_REQUIRE(ub >= 1.0, HS_EINVAL, "METIS API: ubvec must be >= 1");
  const double tol = (ub - 1.0) * *std::min_element(tp.begin(), tp.end());
  const uint64_t seed = opt(kOptSeed) >= 0 ? (uint64_t)opt(kOptSeed) : 0;
  cudaStream_t s = 0;
  std::vector<int64_t> hx(n + 1);
  for (int i = 0; i <= n; ++i) hx[i] = (int64_t)xadj[i] - base;
  for (int i = 0; i < n; ++i)
    HS_REQUIRE(hx[i] <= hx[i + 1], HS_EINVAL, "METIS API: xadj not non-decreasing at %d", i);
  std::vector<int32_t> ha(std::max<int64_t>(nnz, 1), 0);
  for (int64_t j = 0; j < nnz; ++j) {
    const int32_t u = adjncy[j] - base;
    HS_REQUIRE(u >= 0 && u < n, HS_EINVAL, "METIS API: adjncy[%lld] = %d out of range",
               (long long)j, adjncy[j]);
    ha[j] = u;
  }
  std::vector<int32_t> hv(n, 1), hw(std::max<int64_t>(nnz, 1), 1);
  if (vwgt) std::copy(vwgt, vwgt + n, hv.begin());
  if (adjwgt) std::copy(adjwgt, adjwgt + nnz, hw.begin());
  hs::Scratch<int64_t> dx;
  hs::Scratch<int32_t> da, dw, dv, dp;
  HS_CHECK_CUDA(dx.alloc(n + 1, s));
  HS_CHECK_CUDA(da.alloc(std::max<int64_t>(nnz, 1), s));
  HS_CHECK_CUDA(dw.alloc(std::max<int64_t>(nnz, 1), s));
  HS_CHECK_CUDA(dv.alloc(n, s));
  HS_CHECK_CUDA(dp.alloc(n, s));
  HS_CHECK_CUDA(cudaMemcpyAsync(dx, hx.data(), (n + 1) * 8, cudaMemcpyHostToDevice, s));
  if (nnz) {
    HS_CHECK_CUDA(cudaMemcpyAsync(da, ha.data(), nnz * 4, cudaMemcpyHostToDevice, s));
    HS_CHECK_CUDA(cudaMemcpyAsync(dw, hw.data(), nnz * 4, cudaMemcpyHostToDevice, s));
  }
  HS_CHECK_CUDA(cudaMemcpyAsync(dv, hv.data(), n * 4, cudaMemcpyHostToDevice, s));
  hs_ugraph_t g;
  g.n = n;
  g.nnz = nnz;
  g.xadj = dx;
  g.adjncy = da;
  g.adjwgt = nullptr;
  g.adjwgt_i = adjwgt ? (int32_t *)dw : nullptr;  // NULL: unit weights, as in METIS
  g.vwgt = nullptr;
  g.vwgt_i = dv;
  g.twin = nullptr;
  int64_t stats[8] = {0};
  int rc = hs_partition_kway(&g, k, tp.data(), tol, seed, dp, stats, s);
  if (rc) return rc;
  HS_CHECK_CUDA(cudaMemcpyAsync(part, dp, n * 4, cudaMemcpyDeviceToHost, s));
  HS_CHECK_CUDA(cudaStreamSynchronize(s));
  if (base)
    for (int i = 0; i < n; ++i) part[i] += base;
  if (objval) *objval = (int32_t)std::min<int64_t>(stats[0], INT32_MAX);
  return HS_OK;
}
}  // namespace

extern "C" int hs_METIS_PartGraphKway(const int32_t *nvtxs, const int32_t *ncon,
                                      const int32_t *xadj, const int32_t *adjncy,
                                      const int32_t *vwgt, const int32_t *vsize,
                                      const int32_t *adjwgt, const int32_t *nparts,
                                      const float *tpwgts, const float *ubvec,
                                      const int32_t *options, int32_t *objval, int32_t *part) {
  (void)vsize;  // communication volume objective only (METIS_OBJTYPE_VOL)
  const int rc = part_graph_kway(nvtxs, ncon, xadj, adjncy, vwgt, adjwgt, nparts, tpwgts, ubvec,
                                 options, objval, part);
  if (rc == HS_ECUDA && cudaGetLastError() == cudaErrorMemoryAllocation) return kMetisErrorMemory;
  return metis_status(rc);
}

extern "C" int METIS_PartGraphKway(const int32_t *nvtxs, const int32_t *ncon,
                                   const int32_t *xadj, const int32_t *adjncy,
                                   const int32_t *vwgt, const int32_t *vsize,
                                   const int32_t *adjwgt, const int32_t *nparts,
                                   const float *tpwgts, const float *ubvec,
                                   const int32_t *options, int32_t *objval, int32_t *part) {
  return hs_METIS_PartGraphKway(nvtxs, ncon, xadj, adjncy, vwgt, vsize, adjwgt, nparts, tpwgts,
                                ubvec, options, objval, part);
}
