// METIS wire boundary on the device: the reference's
// emit_metis (pkg/src/hetsched/graphio.py:277-304) and parse_partition_file
// (graphio.py:307-330) for graphs far beyond the Python string builders.
//
// emit: the undirected kernel graph (K1 output, integer weights) becomes
//   METIS text: one line per vertex, "vw nbr w nbr w ...", neighbours
//   1-based and ascending (graph.py's sorted((nbr, w))). Row lengths in
//   bytes -> exclusive scan -> one warp per row writes its digits at the
//   scanned offsets (warp scan over the entries' lengths). Byte-bound work.
// parse: partition-file text -> one class per line (empty / 0 / 1 / other
//   integer / not simple), split exactly where Python's str.splitlines
//   splits (\n, \r, \r\n, \v, \f, \x1c-\x1e, U+0085, U+2028, U+2029 in
//   UTF-8) and stripped like str.strip for ASCII whitespace. Lines the
//   device cannot decide (non-ASCII, '_' digit separators, > 18 digits) are
//   reported for the caller to finish with Python's int().
#include "common.cuh"
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <cub/device/device_segmented_sort.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <vector>

namespace {

__device__ __forceinline__ int ndigits(uint32_t x) {
  int d = 1;
  while (x >= 10) { x /= 10; ++d; }
  return d;
}

__device__ __forceinline__ void put_uint(char *out, uint32_t x, int nd) {
  for (int i = nd - 1; i >= 0; --i) { out[i] = (char)('0' + x % 10); x /= 10; }
}

__global__ void seg_bounds_k(int n, const int64_t *xadj, int64_t *b, int64_t *e) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    b[i] = xadj[i];
    e[i] = xadj[i + 1];
  }
}

// bytes of row v: vw, " nbr w" per entry, '\n'
__global__ void row_bytes(int n, const int64_t *xadj, const int32_t *adj, const int32_t *wgt,
                          const int32_t *vw, int64_t *len) {
  const int lane = threadIdx.x & 31;
  const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v = wid; v < n; v += nw) {
    int64_t s = 0;
    for (int64_t j = xadj[v] + lane; j < xadj[v + 1]; j += 32)
      s += 2 + ndigits((uint32_t)adj[j] + 1u) + ndigits((uint32_t)wgt[j]);
    for (int off = 16; off; off >>= 1) s += __shfl_down_sync(0xffffffffu, s, off);
    if (lane == 0) len[v] = s + ndigits((uint32_t)vw[v]) + 1;
  }
}

__global__ void write_rows(int n, const int64_t *xadj, const int32_t *adj, const int32_t *wgt,
                           const int32_t *vw, const int64_t *off, char *text) {
  const int lane = threadIdx.x & 31;
  const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v = wid; v < n; v += nw) {
    char *row = text + off[v];
    const int dv = ndigits((uint32_t)vw[v]);
    if (lane == 0) put_uint(row, (uint32_t)vw[v], dv);
    int64_t pos = dv;  // warp-uniform running position
    for (int64_t j0 = xadj[v]; j0 < xadj[v + 1]; j0 += 32) {
      const int64_t j = j0 + lane;
      const bool ok = j < xadj[v + 1];
      const uint32_t a = ok ? (uint32_t)adj[j] + 1u : 0u, w = ok ? (uint32_t)wgt[j] : 0u;
      const int da = ok ? ndigits(a) : 0, dw = ok ? ndigits(w) : 0;
      const int L = ok ? 2 + da + dw : 0;
      int inc = L;  // inclusive warp scan of the entry lengths
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
      }
      if (ok) {
        char *p = row + pos + inc - L;
        p[0] = ' ';
        put_uint(p + 1, a, da);
        p[1 + da] = ' ';
        put_uint(p + 2 + da, w, dw);
      }
      pos += __shfl_sync(0xffffffffu, inc, 31);
    }
    if (lane == 0) row[pos] = '\n';
  }
}

// ---- partition files --------------------------------------------------------
// Separator starting at byte i (0 = none), its length in *len.
__device__ __forceinline__ bool sep_at(const uint8_t *t, int64_t n, int64_t i, int *len) {
  const uint8_t c = t[i];
  *len = 1;
  if (c == '\n') return i == 0 || t[i - 1] != '\r';  // "\r\n" is one separator
  if (c == '\r') { *len = (i + 1 < n && t[i + 1] == '\n') ? 2 : 1; return true; }
  if (c == 0x0b || c == 0x0c || c == 0x1c || c == 0x1d || c == 0x1e) return true;
  if (c == 0xC2 && i + 1 < n && t[i + 1] == 0x85) { *len = 2; return true; }
  if (c == 0xE2 && i + 2 < n && t[i + 1] == 0x80 && (t[i + 2] == 0xA8 || t[i + 2] == 0xA9)) {
    *len = 3;
    return true;
  }
  return false;
}

__global__ void sep_flags(const uint8_t *t, int64_t n, uint8_t *flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int len;
    flag[i] = sep_at(t, n, i, &len) ? 1 : 0;
  }
}

__device__ __forceinline__ bool ascii_space(uint8_t c) {
  return c == ' ' || (c >= 0x09 && c <= 0x0d) || (c >= 0x1c && c <= 0x1f);
}

// class: 0 empty, 1 -> 0, 2 -> 1, 3 other integer (value in val), 4 undecided
__global__ void classify_lines(const uint8_t *t, int64_t n, const int64_t *seps, int64_t nsep,
                               int8_t *cls, int64_t *val) {
  const int64_t nlines = nsep + 1;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nlines;
       k += (int64_t)gridDim.x * blockDim.x) {
    int64_t s = 0;
    if (k > 0) {
      int len;
      sep_at(t, n, seps[k - 1], &len);
      s = seps[k - 1] + len;
    }
    int64_t e = k < nsep ? seps[k] : n;
    while (s < e && ascii_space(t[s])) ++s;
    while (e > s && ascii_space(t[e - 1])) --e;
    int8_t c = 4;
    int64_t v = 0;
    if (s == e) {
      c = 0;
    } else {
      int64_t i = s;
      bool neg = false;
      if (t[i] == '+' || t[i] == '-') { neg = t[i] == '-'; ++i; }
      bool ok = i < e && e - i <= 18;
      for (int64_t j = i; ok && j < e; ++j) {
        if (t[j] < '0' || t[j] > '9') ok = false;
        else v = v * 10 + (t[j] - '0');
      }
      if (ok) {
        v = neg ? -v : v;
        c = v == 0 ? 1 : (v == 1 ? 2 : 3);
      }
    }
    cls[k] = c;
    val[k] = v;
  }
}

__global__ void line_flags(const int8_t *cls, int64_t nlines, uint8_t *nonempty, uint8_t *odd) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nlines;
       k += (int64_t)gridDim.x * blockDim.x) {
    nonempty[k] = cls[k] != 0;
    odd[k] = cls[k] >= 3;
  }
}

// rank of each odd line among the non-empty lines (its slot in part[])
__global__ void odd_ranks(const int64_t *odd, int64_t k, const int64_t *ne, int64_t nne,
                          int64_t *rank) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = nne;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (ne[mid] < odd[i]) lo = mid + 1; else hi = mid;
    }
    rank[i] = lo;
  }
}

__global__ void gather_values(const int8_t *cls, const int64_t *lines, int64_t count,
                              int8_t *part) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int8_t c = cls[lines[i]];
    part[i] = c == 2 ? 1 : 0;  // classes >= 3 are settled by the caller
  }
}

int select_flagged(int64_t n, const uint8_t *flags, int64_t *out, int64_t *count, cudaStream_t s) {
  thrust::counting_iterator<int64_t> it(0);
  size_t tb = 0;
  HS_CHECK_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, it, flags, out, count, n, s));
  hs::Scratch<char> tmp;
  HS_CHECK_CUDA(tmp.alloc(tb, s));
  HS_CHECK_CUDA(cub::DeviceSelect::Flagged(tmp.p, tb, it, flags, out, count, n, s));
  hs::count_launch(1);
  return HS_OK;
}

}  // namespace

extern "C" int hs_emit_metis(const hs_ugraph_t *g, char *text, int64_t cap, int64_t *len_host,
                             void *stream) {
  HS_REQUIRE(g && len_host && (g->n == 0 || (g->vwgt_i && g->xadj)) &&
                 (g->nnz == 0 || (g->adjncy && g->adjwgt_i)),
             HS_EINVAL, "hs_emit_metis: null argument (needs integer weights)");
  cudaStream_t s = (cudaStream_t)stream;
  const int n = g->n;
  const int64_t nnz = g->nnz;
  // sorted copy of every list (ascending neighbour)
  hs::Scratch<int32_t> adj2, wgt2;
  hs::Scratch<int64_t> b, e, len, off;
  HS_CHECK_CUDA(adj2.alloc(nnz, s));
  HS_CHECK_CUDA(wgt2.alloc(nnz, s));
  HS_CHECK_CUDA(b.alloc(n, s));
  HS_CHECK_CUDA(e.alloc(n, s));
  HS_CHECK_CUDA(len.alloc(n + 1, s));
  HS_CHECK_CUDA(off.alloc(n + 1, s));
  seg_bounds_k<<<hs::grid_for(n, 256), 256, 0, s>>>(n, g->xadj, b, e);
  HS_CHECK_LAUNCH();
  if (nnz > 0) {
    size_t tb = 0;
    HS_CHECK_CUDA(cub::DeviceSegmentedSort::SortPairs(nullptr, tb, g->adjncy, adj2.p, g->adjwgt_i,
                                                      wgt2.p, nnz, n, b.p, e.p, s));
    hs::Scratch<char> tmp;
    HS_CHECK_CUDA(tmp.alloc(tb, s));
    HS_CHECK_CUDA(cub::DeviceSegmentedSort::SortPairs(tmp.p, tb, g->adjncy, adj2.p, g->adjwgt_i,
                                                      wgt2.p, nnz, n, b.p, e.p, s));
    hs::count_launch(2);
  }
  const int wgrid = hs::grid_for((int64_t)n * 32, 256, hs::sm_count() * 32);
  row_bytes<<<wgrid, 256, 0, s>>>(n, g->xadj, adj2, wgt2, g->vwgt_i, len);
  HS_CHECK_LAUNCH();
  HS_CHECK_CUDA(cudaMemsetAsync(len.p + n, 0, sizeof(int64_t), s));
  {
    size_t tb = 0;
    HS_CHECK_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, len.p, off.p, n + 1, s));
    hs::Scratch<char> tmp;
    HS_CHECK_CUDA(tmp.alloc(tb, s));
    HS_CHECK_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, len.p, off.p, n + 1, s));
    hs::count_launch(1);
  }
  int64_t total = 0;
  HS_CHECK_CUDA(cudaMemcpyAsync(&total, off.p + n, 8, cudaMemcpyDeviceToHost, s));
  HS_CHECK_CUDA(cudaStreamSynchronize(s));
  *len_host = total;
  if (!text) return HS_OK;  // size query
  HS_REQUIRE(cap >= total, HS_ELIMIT, "hs_emit_metis: text buffer of %lld bytes < %lld needed",
             (long long)cap, (long long)total);
  {
    hs::Prof P("emit_metis", s, 8.0 * n + 8.0 * nnz + (double)total);
    write_rows<<<wgrid, 256, 0, s>>>(n, g->xadj, adj2, wgt2, g->vwgt_i, off, text);
  }
  HS_CHECK_LAUNCH();
  return HS_OK;
}

extern "C" int hs_parse_partition(const uint8_t *text, int64_t len, int32_t n_expected,
                                  int8_t *part, int64_t *odd_lines, int64_t *odd_values,
                                  int32_t odd_cap, int64_t *info_host, void *stream) {
  HS_REQUIRE(info_host && (len == 0 || text), HS_EINVAL, "hs_parse_partition: null argument");
  cudaStream_t s = (cudaStream_t)stream;
  hs::Scratch<uint8_t> flag;
  hs::Scratch<int64_t> seps, cnt;
  HS_CHECK_CUDA(flag.alloc(len + 1, s));
  HS_CHECK_CUDA(seps.alloc(len + 1, s));
  HS_CHECK_CUDA(cnt.alloc(2, s));
  int64_t nsep = 0;
  if (len > 0) {
    sep_flags<<<hs::grid_for(len, 256), 256, 0, s>>>(text, len, flag);
    HS_CHECK_LAUNCH();
    int rc = select_flagged(len, flag, seps, cnt, s);
    if (rc) return rc;
    HS_CHECK_CUDA(cudaMemcpyAsync(&nsep, cnt, 8, cudaMemcpyDeviceToHost, s));
    HS_CHECK_CUDA(cudaStreamSynchronize(s));
  }
  const int64_t nlines = nsep + 1;
  hs::Scratch<int8_t> cls;
  hs::Scratch<int64_t> val, ne_idx, odd_idx;
  hs::Scratch<uint8_t> ne, odd;
  HS_CHECK_CUDA(cls.alloc(nlines, s));
  HS_CHECK_CUDA(val.alloc(nlines, s));
  HS_CHECK_CUDA(ne.alloc(nlines, s));
  HS_CHECK_CUDA(odd.alloc(nlines, s));
  HS_CHECK_CUDA(ne_idx.alloc(nlines, s));
  HS_CHECK_CUDA(odd_idx.alloc(nlines, s));
  {
    hs::Prof P("parse_partition", s, 3.0 * (double)len + 18.0 * (double)nlines);
    classify_lines<<<hs::grid_for(nlines, 256), 256, 0, s>>>(text, len, seps, nsep, cls, val);
  }
  HS_CHECK_LAUNCH();
  line_flags<<<hs::grid_for(nlines, 256), 256, 0, s>>>(cls, nlines, ne, odd);
  HS_CHECK_LAUNCH();
  int rc = select_flagged(nlines, ne, ne_idx, cnt, s);
  if (rc) return rc;
  rc = select_flagged(nlines, odd, odd_idx, cnt + 1, s);
  if (rc) return rc;
  int64_t c2[2];
  HS_CHECK_CUDA(cudaMemcpyAsync(c2, cnt, 16, cudaMemcpyDeviceToHost, s));
  HS_CHECK_CUDA(cudaStreamSynchronize(s));
  info_host[0] = c2[0];  // non-empty lines
  info_host[1] = c2[1];  // lines the device did not settle to 0/1
  info_host[2] = nlines;
  // odd lines (line index, class, slot in part[]) and values, in line order
  const int64_t k = c2[1] < odd_cap ? c2[1] : odd_cap;
  if (k > 0 && odd_lines && odd_values) {
    hs::Scratch<int64_t> rank;
    HS_CHECK_CUDA(rank.alloc(k, s));
    odd_ranks<<<hs::grid_for(k, 256), 256, 0, s>>>(odd_idx, k, ne_idx, c2[0], rank);
    HS_CHECK_LAUNCH();
    std::vector<int64_t> idx(k), v(k), rk(k);
    std::vector<int8_t> c(k);
    HS_CHECK_CUDA(cudaMemcpyAsync(idx.data(), odd_idx, k * 8, cudaMemcpyDeviceToHost, s));
    HS_CHECK_CUDA(cudaMemcpyAsync(rk.data(), rank.p, k * 8, cudaMemcpyDeviceToHost, s));
    HS_CHECK_CUDA(cudaStreamSynchronize(s));
    for (int64_t i = 0; i < k; ++i) {
      HS_CHECK_CUDA(cudaMemcpyAsync(&c[i], cls.p + idx[i], 1, cudaMemcpyDeviceToHost, s));
      HS_CHECK_CUDA(cudaMemcpyAsync(&v[i], val.p + idx[i], 8, cudaMemcpyDeviceToHost, s));
    }
    HS_CHECK_CUDA(cudaStreamSynchronize(s));
    for (int64_t i = 0; i < k; ++i) {
      odd_lines[3 * i] = idx[i];
      odd_lines[3 * i + 1] = c[i];
      odd_lines[3 * i + 2] = rk[i];
      odd_values[i] = v[i];
    }
  }
  if (part && c2[0] == n_expected) {
    gather_values<<<hs::grid_for(c2[0], 256), 256, 0, s>>>(cls, ne_idx, c2[0], part);
    HS_CHECK_LAUNCH();
  }
  return HS_OK;
}
