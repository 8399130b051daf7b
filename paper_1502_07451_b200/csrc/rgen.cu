// Batched generate_random_dag (pkg/src/hetsched/graph.py:180-305) on the
// device, graph for graph identical to the reference: one thread per graph
// runs CPython's random.Random(seed) — MT19937 seeded by init_by_array with
// the 32-bit words of |seed| (Modules/_randommodule.c), getrandbits(k) =
// genrand_uint32() >> (32 - k), _randbelow by rejection on bit_length(n)
// bits, Random.sample's two strategies (a shrinking pool when the
// population is small, a rejection set otherwise, Lib/random.py) — in the
// reference's draw order:
//   1. when the input slots are not all used: one sample over the slot list
//      (count_root: the kernels' first slots are mandatory, the sample is
//      drawn from their second slots);
//   2. per kernel in id order, sample(earlier kernels, c) for its c inputs;
//   3. sample(unused last-layer sink pairs, extra) for surplus edges;
//   4. root edges to every kernel left without an input.
// The shape (layers, slot counts, targets) depends only on (n, m, layers,
// count_root) and is computed on the host, which also raises the
// reference's InfeasibleGraphError. A second kernel writes each graph's
// out-CSR sorted by (src, dst) and its in-CSR (ascending sources), the
// DagBatch layout of csrc/des.cu.
#include "common.cuh"

namespace {

constexpr int kMtN = 624, kMtM = 397;

struct PyRandom {
  uint32_t *mt;  // word i at mt[i * stride]
  int64_t stride;
  int idx;
  __device__ __forceinline__ uint32_t &at(int i) { return mt[(int64_t)i * stride]; }
  __device__ void init_genrand(uint32_t s) {
    at(0) = s;
    uint32_t prev = s;
    for (int i = 1; i < kMtN; ++i) {
      prev = 1812433253u * (prev ^ (prev >> 30)) + (uint32_t)i;
      at(i) = prev;
    }
    idx = kMtN;
  }
  __device__ void init_by_array(const uint32_t *key, int klen) {
    init_genrand(19650218u);
    int i = 1, j = 0;
    for (int k = kMtN > klen ? kMtN : klen; k; --k) {
      at(i) = (at(i) ^ ((at(i - 1) ^ (at(i - 1) >> 30)) * 1664525u)) + key[j] + (uint32_t)j;
      ++i;
      ++j;
      if (i >= kMtN) {
        at(0) = at(kMtN - 1);
        i = 1;
      }
      if (j >= klen) j = 0;
    }
    for (int k = kMtN - 1; k; --k) {
      at(i) = (at(i) ^ ((at(i - 1) ^ (at(i - 1) >> 30)) * 1566083941u)) - (uint32_t)i;
      ++i;
      if (i >= kMtN) {
        at(0) = at(kMtN - 1);
        i = 1;
      }
    }
    at(0) = 0x80000000u;
    idx = kMtN;
  }
  __device__ uint32_t next() {
    if (idx >= kMtN) {
      const uint32_t mag[2] = {0u, 0x9908b0dfu};
      int kk = 0;
      for (; kk < kMtN - kMtM; ++kk) {
        const uint32_t y = (at(kk) & 0x80000000u) | (at(kk + 1) & 0x7fffffffu);
        at(kk) = at(kk + kMtM) ^ (y >> 1) ^ mag[y & 1u];
      }
      for (; kk < kMtN - 1; ++kk) {
        const uint32_t y = (at(kk) & 0x80000000u) | (at(kk + 1) & 0x7fffffffu);
        at(kk) = at(kk + (kMtM - kMtN)) ^ (y >> 1) ^ mag[y & 1u];
      }
      const uint32_t y = (at(kMtN - 1) & 0x80000000u) | (at(0) & 0x7fffffffu);
      at(kMtN - 1) = at(kMtM - 1) ^ (y >> 1) ^ mag[y & 1u];
      idx = 0;
    }
    uint32_t y = at(idx++);
    y ^= y >> 11;
    y ^= (y << 7) & 0x9d2c5680u;
    y ^= (y << 15) & 0xefc60000u;
    y ^= y >> 18;
    return y;
  }
  // _randbelow_with_getrandbits(n), 0 < n < 2^32
  __device__ uint32_t randbelow(uint32_t n) {
    const int k = 32 - __clz(n);
    uint32_t r = next() >> (32 - k);
    while (r >= n) r = next() >> (32 - k);
    return r;
  }
};

// Random.sample's set size bound (Lib/random.py): 21, plus 4**ceil(log(3k, 4))
// when k > 5; 3k is never a power of 4, so the ceil is the smallest j with
// 4**j > 3k.
__device__ __forceinline__ int64_t sample_setsize(int64_t k) {
  int64_t s = 21;
  if (k > 5) {
    int64_t p = 1;
    while (p <= 3 * k) p *= 4;
    s += p;
  }
  return s;
}

// sample(population, k): population[i] = pop(i) (i < n); result positions
// written through out(i, value). pool: n scratch ints (pool strategy);
// sel: (n + 31) / 32 scratch words (set strategy).
template <class Pop, class Out>
__device__ void py_sample(PyRandom &rng, int64_t n, int64_t k, Pop pop, Out out, int32_t *pool,
                          uint32_t *sel) {
  if (n <= sample_setsize(k)) {
    for (int64_t i = 0; i < n; ++i) pool[i] = pop(i);
    for (int64_t i = 0; i < k; ++i) {
      const int64_t j = rng.randbelow((uint32_t)(n - i));
      out(i, pool[j]);
      pool[j] = pool[n - i - 1];
    }
  } else {
    for (int64_t w = 0; w < (n + 31) / 32; ++w) sel[w] = 0u;
    for (int64_t i = 0; i < k; ++i) {
      int64_t j = rng.randbelow((uint32_t)n);
      while ((sel[j >> 5] >> (j & 31)) & 1u) j = rng.randbelow((uint32_t)n);
      sel[j >> 5] |= 1u << (j & 31);
      out(i, pop(j));
    }
  }
}

struct GenShape {
  int32_t n_real, n_layers;
  const int32_t *first;    // [n_layers + 1]: layer li = kernel ids [first[li], first[li+1])
  int64_t base_capacity;   // slot-list length
  int64_t inter_target, extra;
  int32_t mode;            // 0 all slots used, 1 sample the slots, 2 count_root sample
  int64_t pop_cap;         // pool / bitmap capacity per graph
  int64_t edge_cap;        // edges per graph (scratch)
};


__device__ __forceinline__ int reps_of(const GenShape &S, int li) {
  const int e = S.first[li] - 1;
  return e < 2 ? e : 2;
}

__global__ void rgen_edges(GenShape S, int32_t batch, const int64_t *seeds, uint32_t *mt,
                           int32_t *counts, int32_t *pool, uint32_t *sel, int32_t *lastp,
                           int32_t *esrc, int32_t *edst, int32_t *m_out) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= batch) return;
  PyRandom rng{mt + b, batch, kMtN};
  {
    const int64_t sd = seeds[b];
    const uint64_t a = sd < 0 ? (uint64_t)(-(sd + 1)) + 1 : (uint64_t)sd;
    uint32_t key[2] = {(uint32_t)a, (uint32_t)(a >> 32)};
    rng.init_by_array(key, key[1] ? 2 : 1);
  }
  const int nr = S.n_real;
  int32_t *cnt = counts + (int64_t)b * (nr + 1);
  int32_t *pl = pool + (int64_t)b * S.pop_cap;
  uint32_t *sl = sel + (int64_t)b * ((S.pop_cap + 31) / 32);
  const int L = S.n_layers;
  const int32_t last_lo = S.first[L - 1], last_hi = S.first[L];
  int32_t *lp = lastp + (int64_t)b * 2 * (last_hi - last_lo);  // <= 2 preds per last-layer kernel
  int32_t *es = esrc + (int64_t)b * S.edge_cap, *ed = edst + (int64_t)b * S.edge_cap;
  int64_t m = 0;
  for (int k = 0; k <= nr; ++k) cnt[k] = 0;
  // 1. input counts per kernel
  if (S.mode == 0) {
    for (int li = 1; li < L; ++li)
      for (int k = S.first[li]; k < S.first[li + 1]; ++k) cnt[k] = reps_of(S, li);
  } else {
    // the slot list ([k] * reps per kernel past layer 0) or, count_root, its
    // second slots (list.remove drops each kernel's first occurrence)
    auto slot = [&](int64_t i) -> int32_t {
      int64_t base = 0;  // slots of layers below li
      for (int li = 1; li < L; ++li) {
        const int64_t nk = S.first[li + 1] - S.first[li];
        const int r = reps_of(S, li);
        const int64_t cap = S.mode == 1 ? nk * r : (r == 2 ? nk : 0);
        if (i < base + cap) {
          const int64_t off = i - base;
          return S.first[li] + (int32_t)(S.mode == 1 ? off / r : off);
        }
        base += cap;
      }
      return -1;
    };
    int64_t n_pop = 0, want = S.inter_target;
    for (int li = 1; li < L; ++li) {
      const int64_t nk = S.first[li + 1] - S.first[li];
      const int r = reps_of(S, li);
      n_pop += S.mode == 1 ? nk * r : (r == 2 ? nk : 0);
      if (S.mode == 2)
        for (int k = S.first[li]; k < S.first[li + 1]; ++k) cnt[k] = 1;  // mandatory
    }
    if (S.mode == 2) want -= (nr - (S.first[1] - 1));
    py_sample(rng, n_pop, want, slot, [&](int64_t, int32_t k) { cnt[k] += 1; }, pl, sl);
  }
  // 2. predecessors per kernel, in id order
  for (int li = 1; li < L; ++li) {
    const int32_t ne = S.first[li] - 1;  // earlier kernels: ids 1..ne
    for (int k = S.first[li]; k < S.first[li + 1]; ++k) {
      const int c = cnt[k];
      if (!c) continue;
      py_sample(rng, ne, c, [](int64_t i) -> int32_t { return (int32_t)(1 + i); },
                [&](int64_t i, int32_t u) {
                  es[m] = u;
                  ed[m] = k;
                  ++m;
                  if (li == L - 1) lp[2 * (k - last_lo) + i] = u;
                },
                pl, sl);
      if (li == L - 1 && c < 2) lp[2 * (k - last_lo) + 1] = 0;
    }
  }
  // 3. surplus edges: unused sink pairs (k ascending, u ascending)
  if (S.extra > 0) {
    int64_t nc = 0;
    for (int k = last_lo; k < last_hi; ++k) {
      const int c = cnt[k];
      const int32_t p0 = c > 0 ? lp[2 * (k - last_lo)] : 0, p1 = c > 1 ? lp[2 * (k - last_lo) + 1] : 0;
      for (int32_t u = 1; u < last_lo; ++u)
        if (u != p0 && u != p1) pl[nc++] = (k - last_lo) * last_lo + u;  // encoded pair
    }
    // sample over the encoded list; pool strategy needs its own copy, so
    // move the candidates past the pool region used by py_sample
    int32_t *cand = pl + S.pop_cap / 2;
    for (int64_t i = nc - 1; i >= 0; --i) cand[i] = pl[i];
    py_sample(rng, nc, S.extra, [&](int64_t i) -> int32_t { return cand[i]; },
              [&](int64_t, int32_t code) {
                es[m] = code % last_lo;
                ed[m] = last_lo + code / last_lo;
                ++m;
                cnt[last_lo + code / last_lo] += 1;
              },
              pl, sl);
  }
  // 4. the root feeds every kernel without an input
  for (int k = 1; k <= nr; ++k)
    if (cnt[k] == 0) {
      es[m] = 0;
      ed[m] = k;
      ++m;
    }
  m_out[b] = (int32_t)m;
}

// per graph: out-CSR sorted by (src, dst), in-CSR with ascending sources
__global__ void rgen_csr(int32_t batch, int32_t n, const int64_t *edge_off, const int32_t *esrc,
                         const int32_t *edst, int64_t edge_cap, int64_t *out_ptr,
                         int32_t *out_dst, int64_t *in_ptr, int32_t *in_src, int32_t *in_eid) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= batch) return;
  const int64_t e0 = edge_off[b];
  const int m = (int)(edge_off[b + 1] - e0);
  const int32_t *es = esrc + (int64_t)b * edge_cap, *ed = edst + (int64_t)b * edge_cap;
  int64_t *op = out_ptr + (int64_t)b * (n + 1), *ip = in_ptr + (int64_t)b * (n + 1);
  int32_t *od = out_dst + e0, *is = in_src + e0, *ie = in_eid + e0;
  for (int v = 0; v <= n; ++v) op[v] = 0, ip[v] = 0;
  for (int e = 0; e < m; ++e) {
    op[es[e] + 1] += 1;
    ip[ed[e] + 1] += 1;
  }
  for (int v = 0; v < n; ++v) {
    op[v + 1] += op[v];
    ip[v + 1] += ip[v];
  }
  // fill each source's slots (lists are short), then sort each by destination
  for (int v = 0; v < n; ++v)
    for (int64_t j = op[v]; j < op[v + 1]; ++j) od[j] = -1;
  for (int e = 0; e < m; ++e) {
    const int s = es[e];
    int64_t j = op[s];
    while (od[j] != -1) ++j;
    od[j] = ed[e];
  }
  for (int v = 0; v < n; ++v) {
    const int64_t a = op[v], z = op[v + 1];
    for (int64_t j = a + 1; j < z; ++j) {
      const int32_t x = od[j];
      int64_t i = j - 1;
      while (i >= a && od[i] > x) {
        od[i + 1] = od[i];
        --i;
      }
      od[i + 1] = x;
    }
  }
  // in-CSR: walk the sorted out-order, append to each destination's list
  for (int v = 0; v < n; ++v)
    for (int64_t j = ip[v]; j < ip[v + 1]; ++j) is[j] = -1;
  for (int u = 0; u < n; ++u)
    for (int64_t j = op[u]; j < op[u + 1]; ++j) {
      const int d = od[j];
      int64_t t = ip[d];
      while (is[t] != -1) ++t;
      is[t] = u;
      ie[t] = (int32_t)j;
    }
}

}  // namespace

extern "C" int hs_random_dag_batch(int32_t batch, const int64_t *seeds_dev, int32_t n_real,
                                   int32_t n_layers, const int32_t *first_dev,
                                   int64_t base_capacity, int64_t inter_target, int64_t extra,
                                   int32_t mode, int64_t pop_cap, int64_t edge_cap,
                                   int64_t *edge_counts_host, int64_t *out_ptr, int32_t *out_dst,
                                   int64_t *in_ptr, int32_t *in_src, int32_t *in_eid,
                                   int64_t edge_total_cap, void *stream) {
  HS_REQUIRE(batch >= 0 && n_real >= 1 && n_layers >= 1 && mode >= 0 && mode <= 2, HS_EINVAL,
             "hs_random_dag_batch: bad shape");
  HS_REQUIRE(seeds_dev && first_dev && edge_counts_host, HS_EINVAL,
             "hs_random_dag_batch: null argument");
  HS_REQUIRE(pop_cap < (1ll << 31) && edge_cap < (1ll << 31), HS_ELIMIT,
             "hs_random_dag_batch: graph too large");
  if (batch == 0) return HS_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const int32_t L = n_layers;
  hs::Scratch<uint32_t> mt, sel;
  hs::Scratch<int32_t> counts, pool, lastp, esrc, edst, m_dev;
  int32_t first_last[2];
  HS_CHECK_CUDA(cudaMemcpyAsync(first_last, first_dev + L - 1, 2 * sizeof(int32_t),
                                cudaMemcpyDeviceToHost, s));
  HS_CHECK_CUDA(cudaStreamSynchronize(s));
  const int64_t n_last = first_last[1] - first_last[0];
  HS_CHECK_CUDA(mt.alloc((int64_t)kMtN * batch, s));
  HS_CHECK_CUDA(counts.alloc((int64_t)batch * (n_real + 1), s));
  HS_CHECK_CUDA(pool.alloc((int64_t)batch * pop_cap, s));
  HS_CHECK_CUDA(sel.alloc((int64_t)batch * ((pop_cap + 31) / 32), s));
  HS_CHECK_CUDA(lastp.alloc((int64_t)batch * 2 * (n_last > 0 ? n_last : 1), s));
  HS_CHECK_CUDA(esrc.alloc((int64_t)batch * edge_cap, s));
  HS_CHECK_CUDA(edst.alloc((int64_t)batch * edge_cap, s));
  HS_CHECK_CUDA(m_dev.alloc(batch, s));
  GenShape S{n_real, n_layers, first_dev, base_capacity, inter_target, extra, mode, pop_cap,
             edge_cap};
  rgen_edges<<<(batch + 63) / 64, 64, 0, s>>>(S, batch, seeds_dev, mt, counts, pool, sel, lastp,
                                               esrc, edst, m_dev);
  HS_CHECK_LAUNCH();
  std::vector<int32_t> mh(batch);
  HS_CHECK_CUDA(cudaMemcpyAsync(mh.data(), m_dev, batch * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  HS_CHECK_CUDA(cudaStreamSynchronize(s));
  std::vector<int64_t> off(batch + 1, 0);
  for (int b = 0; b < batch; ++b) {
    edge_counts_host[b] = mh[b];
    off[b + 1] = off[b] + mh[b];
  }
  if (!out_ptr) return HS_OK;  // sizes only
  HS_REQUIRE(off[batch] <= edge_total_cap, HS_EINVAL,
             "hs_random_dag_batch: edge arrays hold %lld, need %lld", (long long)edge_total_cap,
             (long long)off[batch]);
  hs::Scratch<int64_t> off_dev;
  HS_CHECK_CUDA(off_dev.alloc(batch + 1, s));
  HS_CHECK_CUDA(cudaMemcpyAsync(off_dev, off.data(), (batch + 1) * sizeof(int64_t),
                                cudaMemcpyHostToDevice, s));
  rgen_csr<<<(batch + 63) / 64, 64, 0, s>>>(batch, n_real + 1, off_dev, esrc, edst, edge_cap,
                                             out_ptr, out_dst, in_ptr, in_src, in_eid);
  HS_CHECK_LAUNCH();
  HS_CHECK_CUDA(cudaStreamSynchronize(s));  // the host copy of off goes out of scope
  return HS_OK;
}
